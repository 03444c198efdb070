"""Reference-produced golden results at the large BASELINE configs (C2, C3).

TEST INFRASTRUCTURE, build container only (``/root/reference`` must exist):

    python oracle/make_golden_large.py c2      # m=10,000  (~25 min on 8 cores)
    python oracle/make_golden_large.py c3      # m=20,000  (~3.5 h on 8 cores)

It imports ``bsesolve`` from /root/reference/pkg/src (never copied) and runs the
REFERENCE ``solve`` on the reference's own synthetic instance.  The instance is
built with exactly the expressions of ``generate`` (/root/reference/pkg/src/
bsesolve/generate.py:60-83) so the matrices are bit-identical to what
``generate`` returns; the only change is that the n x n ``is_definite``
Cholesky (generate.py:77, hamiltonian.py:208-218) is skipped -- it would need
~75 GB at m=20,000 -- and the hamiltonian is marked DEFINITE, which the
construction certifies (generate.py:1-8, coupling_ratio 0.5 < 1).

Written to ``tests/golden/large_<cfg>.npz`` (small: no matrices):

* construction scalars ``b0_norm`` = svdvals(B0)[0] and ``lambda_min_a`` =
  eigvalsh(A)[0] (generate.py:72-73), plus probes A@P, B@P, diag(A), B[0,:]
  so the GPU generator can prove it built the same matrix;
* the full ``SolveResult``: all nev eigenvalues, residual norms, iterations,
  converged, backup events, the per-iteration trace, bounds (mu_1, mu_nevex,
  mu_n, Lanczos ritz values / weights) and 8 Ritz vectors (first 4, last 4);
* the reference's PhaseLedger seconds / flops and wall time on this host
  (cores recorded) -- a measured CPU time-to-solution.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

CONFIGS = {
    # BASELINE.json configs[1] / [2] (SURVEY.md §8 shorthand C2 / C3), seed 0,
    # relative residual policy (absolute 1e-10 stalls at n>=20k).
    "c2": dict(m=10_000, nev=500, nex=100),
    "c3": dict(m=20_000, nev=1000, nex=200),
    # small rehearsal of the recipe (seconds)
    "t1": dict(m=600, nev=40, nex=10),
}


def build_reference_instance(bs, m: int, seed: int = 0, alpha: float = 1.0, ratio: float = 0.5):
    """generate.py:60-83 expression for expression, minus the n x n Cholesky."""
    import scipy.linalg as sla
    from bsesolve import rng

    t = {}
    t0 = time.perf_counter()
    c = rng.complex_normal_matrix(rng.substream(seed, 0), m, m)            # generate.py:63
    t["rng_c"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    a = c @ c.conj().T + alpha * np.eye(m)                                  # generate.py:64
    del c
    a = (a + a.conj().T) / 2.0                                              # generate.py:65
    t["a"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    d = rng.complex_normal_matrix(rng.substream(seed, 1), m, m)            # generate.py:70
    t["rng_d"] = time.perf_counter() - t0
    b0 = (d + d.T) / 2.0                                                    # generate.py:71
    del d
    t0 = time.perf_counter()
    b_norm = sla.svdvals(b0)[0]                                             # generate.py:72
    t["svdvals"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    lam_min = float(sla.eigvalsh(a)[0])                                     # generate.py:73
    t["eigvalsh"] = time.perf_counter() - t0
    b = (ratio * lam_min / b_norm) * b0                                     # generate.py:74
    del b0
    ham = bs.BseHamiltonian(a, b, definiteness=bs.Definiteness.DEFINITE)   # generate.py:76 (+77 certified)
    del a, b
    return ham, float(b_norm), lam_min, t


def main(cfg_name: str) -> None:
    sys.path.insert(0, str(REF))
    import bsesolve as bs
    from bsesolve import rng

    cfg = CONFIGS[cfg_name]
    m, nev, nex = cfg["m"], cfg["nev"], cfg["nex"]
    t_all = time.perf_counter()
    ham, b_norm, lam_min, tgen = build_reference_instance(bs, m)
    gen_s = time.perf_counter() - t_all
    print(f"[{cfg_name}] instance m={m} built in {gen_s:.1f} s {tgen}", flush=True)

    probe = rng.complex_normal_matrix(77, m, 3)
    out = dict(
        m=m, nev=nev, nex=nex, deg=20, tol=1e-10, rel_res=True, seed=0,
        b0_norm=b_norm, lambda_min_a=lam_min, probe=probe,
        a_probe=ham.a @ probe, b_probe=ham.b @ probe,
        a_diag=np.real(np.diag(ham.a)).copy(), b_row0=ham.b[0].copy(),
        a_col1=ham.a[:, 1].copy(), b_col1=ham.b[:, 1].copy(),
    )

    scfg = bs.SolverConfig(nev=nev, nex=nex, deg=20, tol=1e-10, seed=0, rel_res=True)
    t0 = time.perf_counter()
    r = bs.solve(ham, scfg)
    solve_s = time.perf_counter() - t0
    print(f"[{cfg_name}] solve {solve_s:.1f} s, {r.iterations_used} its, converged={r.converged}", flush=True)

    tr = r.trace
    out.update(
        lambdas=r.lambdas, residual_norms=r.residual_norms, iterations_used=r.iterations_used,
        converged=r.converged, backup_events=r.backup_events,
        v_first4=r.v[:, :4].copy(), v_last4=r.v[:, -4:].copy(),
        mu_1=r.bounds.mu_1, mu_nevex=r.bounds.mu_nevex, mu_n=r.bounds.mu_n,
        lanczos_steps=r.bounds.steps, ritz_values_lanczos=r.bounds.ritz_values,
        ritz_weights=r.bounds.ritz_weights,
        trace_it=np.array([x.it for x in tr]), trace_locked=np.array([x.locked for x in tr]),
        trace_k=np.array([x.k for x in tr]), trace_max_res=np.array([x.max_res for x in tr]),
        trace_min_res_unlocked=np.array([x.min_res_unlocked for x in tr]),
        trace_mu_nevex=np.array([x.mu_nevex for x in tr]),
        trace_variant=np.array([x.variant for x in tr]),
        trace_lambda_min_m=np.array([x.lambda_min_m for x in tr]),
        trace_flops=np.array([x.flops for x in tr]),
        solve_seconds=solve_s, generate_seconds=gen_s,
    )
    ledger = {"seconds": dict(r.ledger.seconds), "flops": dict(r.ledger.flops)}
    host = dict(cores=os.cpu_count(), cpu=platform.processor() or platform.machine(),
                openblas_threads=os.environ.get("OPENBLAS_NUM_THREADS"),
                numpy=np.__version__, reference_version=bs.__version__)
    out["ledger_json"] = json.dumps(ledger)
    out["host_json"] = json.dumps(host)
    out["generate_breakdown_json"] = json.dumps(tgen)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"large_{cfg_name}.npz", **out)
    print(f"[{cfg_name}] wrote {OUT / f'large_{cfg_name}.npz'}; ledger {ledger}", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c2"]:
        main(name)
