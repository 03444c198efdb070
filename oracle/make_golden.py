"""Generate golden fixtures from the REFERENCE package (build container only).

Run here, where /root/reference exists:

    python oracle/make_golden.py

It imports ``bsesolve`` from /root/reference/pkg/src (read-only, never copied)
and writes small ``.npz`` fixtures under ``tests/golden/``.  The GPU box has no
/root/reference; it only reads the committed fixtures.  TEST INFRASTRUCTURE.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _trace_arrays(trace):
    return {
        "trace_it": np.array([r.it for r in trace]),
        "trace_locked": np.array([r.locked for r in trace]),
        "trace_k": np.array([r.k for r in trace]),
        "trace_max_res": np.array([r.max_res for r in trace]),
        "trace_min_res_unlocked": np.array([r.min_res_unlocked for r in trace]),
        "trace_mu_nevex": np.array([r.mu_nevex for r in trace]),
        "trace_variant": np.array([r.variant for r in trace]),
        "trace_lambda_min_m": np.array([r.lambda_min_m for r in trace]),
        "trace_flops": np.array([r.flops for r in trace]),
    }


def main() -> None:
    sys.path.insert(0, str(REF))
    import bsesolve as bs
    from bsesolve import rng

    OUT.mkdir(parents=True, exist_ok=True)
    meta = {"reference_version": bs.__version__, "numpy": np.__version__}

    # ---- rng (test_rng.py:6-37 published + extra vectors) -------------------
    np.savez(
        OUT / "rng.npz",
        words_seed0=np.array([rng.word(0, i) for i in range(16)], dtype=np.uint64),
        words_deadbeef=np.array([rng.word(0xDEADBEEF, i) for i in range(16)], dtype=np.uint64),
        substreams=np.array([rng.substream(s, t) for s in (0, 1, 42, 2**63) for t in range(4)], dtype=np.uint64),
        normals_12345=rng.complex_normals(12345, 64),
        normals_sub03=rng.complex_normals(rng.substream(0, 3), 257, start_index=5),
        matrix_7_5_3=rng.complex_normal_matrix(7, 5, 3),
    )

    # ---- small instances + sub-operator outputs -----------------------------
    small = {}
    for m, seed in [(8, 11), (16, 5), (24, 100), (32, 4), (32, 6), (32, 8), (32, 14), (32, 15),
                    (32, 16), (48, 12), (48, 13), (64, 21), (64, 40)]:
        cr = 0.0 if (m, seed) == (64, 40) else 0.5
        ham = bs.generate(bs.GeneratorSpec(m=m, seed=seed, coupling_ratio=cr))
        small[f"m{m}_s{seed}"] = ham
        np.savez(OUT / f"ham_m{m}_s{seed}.npz", a=ham.a, b=ham.b)

    ham = small["m16_s5"]
    x = rng.complex_normal_matrix(99, ham.n, 5)
    bounds = bs.estimate_bounds(ham, nevex=6, steps=16, seed=2)
    fcfg = bs.FilterConfig.from_bounds(bounds, 14)
    filt = bs.chebyshev_filter(ham, x, fcfg)
    q, method = bs.cholqr_with_fallback(filt)
    ritz, red = bs.build_hermitian_rq(ham, q)
    res = bs.residuals(ham, ritz)
    ritz_b, red_b = bs.build_backup_rq(ham, q)
    bs.residuals(ham, ritz_b)
    np.savez(
        OUT / "ops_m16_s5.npz",
        x=x, hx=bs.apply_h(ham, x), hx_adj=bs.apply_h_via_adjoint(ham, x),
        mu_1=bounds.mu_1, mu_nevex=bounds.mu_nevex, mu_n=bounds.mu_n, steps=bounds.steps,
        ritz_values_lanczos=bounds.ritz_values, ritz_weights=bounds.ritz_weights,
        deg=14, center=fcfg.center, half_width=fcfg.half_width, scale_ref=fcfg.scale_ref,
        filtered=filt, q=q, method=method,
        rr_values=ritz.values, rr_vectors=ritz.vectors, rr_res=res, rr_lambda_min_m=red.lambda_min_m,
        rr_w=red.w, rr_m=red.m, rr_g=red.g,
        bk_values=ritz_b.values, bk_res=ritz_b.residual_norms,
    )

    # ---- solves on small instances (tests mirror test_solver.py) -----------
    cases = {
        "m64_s21": dict(nev=8, seed=21),
        "m32_s4": dict(nev=4, seed=9),
        "m32_s6": dict(nev=4, seed=6, rr_variant="backup"),
        "m32_s8": dict(nev=4, seed=8, maxiter=1, deg=2),
        "m32_s14": dict(nev=4, seed=14, rel_res=True),
        "m48_s12": dict(nev=6, seed=12),
        "m48_s13": dict(nev=6, seed=13),
        "m64_s40": dict(nev=8, seed=40),
        "m24_s100": dict(nev=3, seed=0),
    }
    solves = {}
    for key, kw in cases.items():
        r = bs.solve(small[key], bs.SolverConfig(**kw))
        eig = bs.direct_solve_definite(small[key]).lambdas
        np.savez(
            OUT / f"solve_{key}.npz",
            lambdas=r.lambdas, v=r.v, residual_norms=r.residual_norms,
            iterations_used=r.iterations_used, converged=r.converged,
            backup_events=r.backup_events, mu_1=r.bounds.mu_1, mu_nevex=r.bounds.mu_nevex,
            dense_lambdas=eig, **_trace_arrays(r.trace),
        )
        solves[key] = kw

    # ---- C1: m=500 seed 0 (BASELINE.json configs[0]) -----------------------
    from bsesolve import fileio
    spec = bs.GeneratorSpec(m=500, seed=0)
    ham = bs.generate(spec)
    # construction scalars so the instance can be rebuilt without the reference
    import scipy.linalg as sla
    d = rng.complex_normal_matrix(rng.substream(0, 1), 500, 500)
    b0 = (d + d.T) / 2.0
    probe = rng.complex_normal_matrix(77, 500, 3)
    c1 = dict(
        b0_norm=sla.svdvals(b0)[0], lambda_min_a=float(sla.eigvalsh(ham.a)[0]),
        a_probe=ham.a @ probe, b_probe=ham.b @ probe, probe=probe,
        a_diag=np.real(np.diag(ham.a)).copy(), b_exact_row0=ham.b[0].copy(),
    )
    tmp = Path("/tmp/c1.pchb")
    fileio.write_pchb(tmp, ham)
    meta["c1_pchb_digest"] = fileio.digest64(tmp)
    for tag, kw in {"abs": dict(rel_res=False), "rel": dict(rel_res=True)}.items():
        r = bs.solve(ham, bs.SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0, **kw))
        c1.update({
            f"{tag}_lambdas": r.lambdas, f"{tag}_res": r.residual_norms,
            f"{tag}_v10": r.v[:, :10], f"{tag}_iters": r.iterations_used,
            f"{tag}_converged": r.converged, f"{tag}_mu_1": r.bounds.mu_1,
            f"{tag}_mu_nevex": r.bounds.mu_nevex,
            f"{tag}_filter_flops": r.ledger.flops["filter"],
            **{f"{tag}_{k}": v for k, v in _trace_arrays(r.trace).items()},
        })
    np.savez(OUT / "c1_m500_s0.npz", **c1)
    meta["cases"] = solves

    # ---- file formats (FORMATS.md): reference writer outputs on small data -------------------
    ham8 = small["m8_s11"]
    fileio.write_pchb(OUT / "m8_s11.pchb", ham8)
    fileio.write_matrix_market(OUT / "m8_s11_A.mtx", ham8.a, comment=" resonant block, seed=11")
    r = bs.solve(small["m32_s4"], bs.SolverConfig(nev=4, seed=9))
    fileio.write_eigenvalues_csv(OUT / "m32_s4_eigenvalues.csv", r.lambdas, r.residual_norms, "0123456789abcdef",
                                 converged=r.converged)
    fileio.write_trace_csv(OUT / "m32_s4_trace.csv", r, "0123456789abcdef")
    fileio.write_pchv(OUT / "m32_s4_v.pchv", r.v)
    np.savez(OUT / "m32_s4_result.npz", lambdas=r.lambdas, res=r.residual_norms, mu_1=r.bounds.mu_1,
             mu_n=r.bounds.mu_n, converged=r.converged, **_trace_arrays(r.trace))
    meta["m8_s11_pchb_digest"] = fileio.digest64(OUT / "m8_s11.pchb")
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
