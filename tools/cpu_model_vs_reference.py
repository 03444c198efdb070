"""The CPU phase model (oracle/cpu_model.py) against the REFERENCE's own measured solve
(tests/golden/large_<cfg>.npz, oracle/make_golden_large.py) on the same host (build container).

    python tools/cpu_model_vs_reference.py c3

Calibrates on a same-shaped definite instance (BLAS time does not depend on the values), evaluates
the model over the reference's own trace and compares phase by phase with the reference's
PhaseLedger seconds.  Writes profiles/r02/cpu_model_vs_reference_<cfg>_container.json."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import cpu_model  # noqa: E402


def main(cfg):
    g = np.load(ROOT / "tests" / "golden" / f"large_{cfg}.npz", allow_pickle=False)
    m, nev, nex = int(g["m"]), int(g["nev"]), int(g["nex"])
    tk, tl = [int(x) for x in g["trace_k"]], [int(x) for x in g["trace_locked"]]
    t0 = time.perf_counter()
    a, b = cpu_model.timing_instance(m)
    cal = cpu_model.calibrate(a, b, nev + nex, min(tk), nev)
    mod = cpu_model.model(cal, tk, tl, int(g["deg"]), int(g["lanczos_steps"]), nevex=nev + nex)
    led = json.loads(str(g["ledger_json"]))["seconds"]
    out = {"cfg": cfg, "reference_solve_s": float(g["solve_seconds"]), "reference_phases_s": led,
           "reference_host": json.loads(str(g["host_json"])), "model_s": mod["total"], "model_phases_s": mod,
           "ratio_model_over_reference": mod["total"] / float(g["solve_seconds"]), "calibration": cal,
           "wall_s": time.perf_counter() - t0,
           "note": "the reference run shared the container's 8 cores with other jobs part of the time"}
    (ROOT / "profiles" / "r02" / f"cpu_model_vs_reference_{cfg}_container.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: out[k] for k in ("reference_solve_s", "model_s", "ratio_model_over_reference")}))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c3")
