"""Check the CPU time-to-solution model (oracle/cpu_model.py) against a MEASURED full solve.

    python tools/cpu_model_check.py c2 [--where box]       (GPU box: builds the input on the GPU)

Builds the config's instance with the GPU generator (the reference construction, tests/
test_gpu_large_parity.py pins it), copies A, B to the host, runs the oracle's complete solve
(bse_oracle.oracle_solve: the reference's numpy / OpenBLAS code path) on all host cores with
per-phase wall seconds, then calibrates the phase model on the same host (full and quick widths)
and evaluates it over the measured solve's own trace.  Writes
profiles/r02/cpu_model_check_<cfg>.json.  The oracle's result is also compared with the
reference's golden result (tests/golden/large_<cfg>.npz) when present.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CONFIGS = {"c2": (10000, 500, 100), "c3": (20000, 1000, 200), "t": (2000, 100, 20)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", choices=sorted(CONFIGS))
    ap.add_argument("--where", default="box")
    args = ap.parse_args()
    m, nev, nex = CONFIGS[args.cfg]
    import torch

    import paper_2601_10557_b200 as bse
    from oracle import bse_oracle as o
    from oracle import cpu_model

    ham = bse.generate(bse.GeneratorSpec(m=m, seed=0), device=torch.device("cuda", 0))
    a, b = ham.host_blocks()
    a, b = np.asfortranarray(a), np.asfortranarray(b)
    ham.release_device()
    del ham
    torch.cuda.empty_cache()
    sec = {}
    t0 = time.perf_counter()
    r = o.oracle_solve(a, b, nev=nev, nex=nex, deg=20, tol=1e-10, seed=0, rel_res=True, seconds=sec)
    wall = time.perf_counter() - t0
    tk = [t["k"] for t in r.trace]
    tl = [t["locked"] for t in r.trace]
    print(f"measured {wall:.1f} s, {r.iterations_used} its, phases {sec}", flush=True)
    nevex = nev + nex
    full = cpu_model.calibrate(a, b, nevex, min(tk), nev)
    quick = cpu_model.calibrate(a, b, min(nevex, 512), 64, min(nev, 256))
    mf = cpu_model.model(full, tk, tl, 20, r.bounds.steps, nevex=nevex)
    mq = cpu_model.model(quick, tk, tl, 20, r.bounds.steps, nevex=nevex)
    out = {"cfg": args.cfg, "where": args.where, "cores": cpu_model._cores(), "measured_s": wall,
           "measured_phases_s": sec, "iterations": r.iterations_used, "trace_k": tk, "trace_locked": tl,
           "model_s": mf["total"], "model_phases_s": mf, "ratio": mf["total"] / wall,
           "quick_model_s": mq["total"], "quick_model_phases_s": mq, "quick_ratio": mq["total"] / wall,
           "calibration_full": full, "calibration_quick": quick}
    g = ROOT / "tests" / "golden" / f"large_{args.cfg}.npz"
    if g.exists():
        gz = np.load(g, allow_pickle=False)
        out["oracle_vs_reference"] = {
            "max_dlambda_rel": float(np.max(np.abs(r.lambdas - gz["lambdas"]) / np.abs(gz["lambdas"]))),
            "iterations": r.iterations_used, "iterations_ref": int(gz["iterations_used"]),
            "trace_locked_equal": tl == [int(x) for x in gz["trace_locked"]],
            "reference_solve_s_build_container": float(gz["solve_seconds"]),
            "reference_host": json.loads(str(gz["host_json"]))}
    dst = ROOT / "profiles" / "r02"
    dst.mkdir(parents=True, exist_ok=True)
    (dst / f"cpu_model_check_{args.cfg}.json").write_text(json.dumps(out, indent=1) + "\n")
    gdst = ROOT / "gpurun_out" / "r02"
    gdst.mkdir(parents=True, exist_ok=True)
    (gdst / f"cpu_model_check_{args.cfg}.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: out[k] for k in ("measured_s", "model_s", "ratio", "quick_model_s", "quick_ratio")}))


if __name__ == "__main__":
    main()
