"""CPU time-to-solution of the reference solver, built from TIMED reference-path phases.

TEST / BENCH INFRASTRUCTURE ONLY (imported by bench.py's ``--impl reference``
arm and its ``cpu_baseline`` leg, and by tools/cpu_model_check.py).  A full
reference solve at the headline config takes hours on the host cores
(C2 = 1,058 s on 8 cores; C3 is ~8x the filter work), so the
bench times each phase of the reference's code path ONCE at the workload's
full n on the box's cores -- the same numpy / OpenBLAS calls the reference
makes, through the oracle restatement (bse_oracle.py) -- and evaluates the
solve's per-iteration work (k active, l locked per outer iteration; the
trace, identical between the reference and the GPU solver, tests/
test_gpu_large_parity.py) against those timings:

  filter    deg * step(k)          step = one recurrence step with the reference's
                                   numpy temporaries, plain and adjoint products
                                   alternating (chebyshev.py:62-74, hamiltonian.py:132-176);
                                   step(k) = s0 + s1 k fitted through k_lo, k_hi
  ortho     qr(l) + proj(l, k) + chol(k)
                                   Householder QR of S Y_locked (ortho.py:149-150, ~ l^2),
                                   projection (ortho.py:151-152, ~ l k), CholQR2 + phase
                                   fix (ortho.py:96-129, c1 k + c2 k^2 through k_lo, k_hi)
  rr        r1 k + r2 k^2          build_hermitian_rq (rayleigh_ritz.py:98-143) timed at
                                   k_lo and k_hi (one H application + n k^2 + k^3 work)
  residuals res(k_lo)/step(k_lo) * step(k)
                                   residuals (rayleigh_ritz.py:182-190): one H application
  lanczos   steps * one Lanczos step (lanczos.py:53-88, k = 1)
  start     the n x nevex start-block draw (solver.py:139-141)

The model is checked against MEASURED full solves: the reference's own C3
solve in the build container (oracle/make_golden_large.py, 8 cores) and the
oracle's C2 solve on the GPU box's 16 cores (profiles/r02/cpu_model_check_*.json).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import bse_oracle as o


def _now():
    return time.perf_counter()


def _block(seed, n, k):
    return o.gauss_c_matrix(seed, n, k)


REPS = 3  # every phase is timed REPS times and the median kept


def _best(fn, reps=REPS):
    ts = []
    for _ in range(reps):
        t0 = _now()
        fn()
        ts.append(_now() - t0)
    return float(np.median(ts))


def _filter_steps(a, b, k, c, e, s):
    """Recurrence steps with the plain and the adjoint product (chebyshev.py:62-74); seconds per
    step (median of REPS pairs)."""
    n = 2 * a.shape[0]
    st = {"y_old": _block(11, n, k), "y": _block(12, n, k), "sig": e / (s - c)}
    sig1 = e / (s - c)

    def pair():
        for prod in (o.h_times, o.h_times_adjoint):
            sn = 1.0 / (2.0 / sig1 - st["sig"])
            y_new = (2.0 * sn / e) * (prod(a, b, st["y"]) - c * st["y"]) - (st["sig"] * sn) * st["y_old"]
            st["y_old"], st["y"], st["sig"] = st["y"], y_new / np.abs(y_new).max(), sn

    return _best(pair) / 2.0


def _orthonormal(n, k, seed):
    q, _ = o.cholqr2(_block(seed, n, k))
    return q


def calibrate(a, b, k_hi: int, k_lo: int, l_hi: int, *, bounds=(-1.0, 0.5, 1.0), reps: int | None = None) -> dict:
    """Time every reference phase at the workload's full n (a, b: host blocks, F-order); each timing
    is the median of `reps` (default REPS) runs."""
    global REPS
    saved = REPS
    REPS = reps or REPS
    try:
        return _calibrate(a, b, k_hi, k_lo, l_hi, bounds)
    finally:
        REPS = saved


def _calibrate(a, b, k_hi, k_lo, l_hi, bounds):
    m = a.shape[0]
    n = 2 * m
    mu_1, cut, mu_n = bounds
    c, e = (mu_n + cut) / 2.0, (mu_n - cut) / 2.0
    t = {"n": n, "k_hi": k_hi, "k_lo": k_lo, "l_hi": l_hi, "cores": _cores(), "reps": REPS,
         "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}
    o.h_times(a, b, _block(1, n, min(k_lo, 64)))  # BLAS threads and buffers up at the full size
    t0 = _now()
    for k in (k_lo, k_hi):
        t[f"step_{k}"] = _filter_steps(a, b, k, c, e, mu_1)
    t1 = _now()
    v_hi = _block(21, n, k_hi)  # the start block draw (solver.py:139-141), per column
    t["start_per_col"] = (_now() - t1) / k_hi
    # ortho pieces (ortho.py:132-158)
    v_lo = _block(22, n, k_lo)
    locked = _orthonormal(n, l_hi, 23)
    res = {}
    t["qr_l"] = _best(lambda: res.__setitem__("basis", np.linalg.qr(o.s_flip(locked))[0]))
    basis = res["basis"]
    t["proj_l_khi"] = _best(lambda: v_hi - basis @ (basis.conj().T @ v_hi))
    for k, v in ((k_lo, v_lo), (k_hi, v_hi)):
        t[f"chol_{k}"] = _best(lambda: o.cholqr2(v))
    del basis, locked, res
    # Rayleigh-Ritz (rayleigh_ritz.py:98-143) and residuals (:182-190)
    for k, v in ((k_lo, v_lo), (k_hi, v_hi)):
        q, _ = o.cholqr2(v)
        out = {}
        t[f"rr_{k}"] = _best(lambda: out.__setitem__("rr", o.rr_hermitian(a, b, q)))
        if k == k_lo:
            lam, vec, _ = out["rr"]
            t[f"res_{k}"] = _best(lambda: o.residual_norms(a, b, lam, vec))
    # Lanczos: one step = one k = 1 H application + S-dots (lanczos.py:53-88)
    x = _block(31, n, 1)[:, 0]
    t["lanczos_step"] = _best(lambda: float(np.real(np.vdot(o.s_flip(o.h_times(a, b, x)), x))), 3)
    t["calibration_s"] = _now() - t0
    return t


def _lin(x0, y0, x1, y1):
    """(intercept, slope) through two points; slope >= 0."""
    slope = max((y1 - y0) / (x1 - x0), 0.0) if x1 != x0 else 0.0
    return y1 - slope * x1, slope


def _quad(x0, y0, x1, y1):
    """y = c1 x + c2 x^2 through two points (no intercept), clipped to c1, c2 >= 0."""
    det = x0 * x1 * x1 - x1 * x0 * x0
    c1 = (y0 * x1 * x1 - y1 * x0 * x0) / det
    c2 = (x0 * y1 - x1 * y0) / det
    if c2 < 0:
        return y1 / x1, 0.0
    if c1 < 0:
        return 0.0, y1 / (x1 * x1)
    return c1, c2


def model(cal: dict, trace_k, trace_locked, deg: int, lanczos_steps: int, step_scale: float = 1.0,
          nevex: int | None = None) -> dict:
    """Per-phase seconds of the reference solve whose iterations had active widths trace_k and
    locked counts trace_locked (after each iteration); step_scale rescales the H-application rate
    from a fresh per-step sample."""
    klo, khi, lhi = cal["k_lo"], cal["k_hi"], cal["l_hi"]
    s0, s1 = _lin(klo, cal[f"step_{klo}"], khi, cal[f"step_{khi}"])
    c1, c2 = _quad(klo, cal[f"chol_{klo}"], khi, cal[f"chol_{khi}"])
    r1, r2 = _quad(klo, cal[f"rr_{klo}"], khi, cal[f"rr_{khi}"])
    res_ratio = cal[f"res_{klo}"] / cal[f"step_{klo}"]
    qr2 = cal["qr_l"] / (lhi * lhi)
    pj = cal["proj_l_khi"] / (lhi * khi)
    out = {"lanczos": lanczos_steps * cal["lanczos_step"] * step_scale, "filter": 0.0, "ortho": 0.0, "rr": 0.0,
           "residuals": 0.0}
    l_before = 0
    for k, l_after in zip(trace_k, trace_locked):
        step = (s0 + s1 * k) * step_scale
        out["filter"] += deg * step
        out["ortho"] += (qr2 * l_before * l_before + pj * l_before * k if l_before else 0.0) + c1 * k + c2 * k * k
        out["rr"] += r1 * k + r2 * k * k
        out["residuals"] += res_ratio * step
        l_before = l_after
    out["start"] = cal["start_per_col"] * (nevex or trace_k[0])
    out["total"] = sum(out.values())
    return out


def sample_step(a, b, k: int) -> float:
    """A bounded per-bench-step sample: one plain H application with the recurrence arithmetic
    (median of REPS)."""
    n = 2 * a.shape[0]
    y = _block(41, n, k)
    y_old = _block(42, n, k)
    return _best(lambda: 0.5 * (o.h_times(a, b, y) - 0.25 * y) - 0.125 * y_old)


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def timing_instance(m: int, seed: int = 12345):
    """Same-shaped definite blocks for timing on a host without the GPU-built input:
    A = (Z + Z^H)/2 + 8 sqrt(m) I, B = 0.05 (Z + Z^T) (S H definite: ||B|| << lambda_min(A)).
    BLAS / LAPACK time does not depend on the values; definiteness keeps the RR's Cholesky
    on the reference's normal path."""
    z = np.asfortranarray(o.gauss_c(seed, m * m).reshape(m, m))
    a = (z + z.conj().T) * 0.5
    a[np.diag_indices(m)] += 8.0 * np.sqrt(m)
    b = np.asfortranarray((z + z.T) * 0.05)
    return np.asfortranarray(a), b


def reference_trace(golden_npz=None, own_json=None):
    """(k per iteration, locked after each iteration, lanczos steps, source) of the solve to model:
    the REFERENCE's own trace (tests/golden/large_<cfg>.npz) when present, else the GPU solve's
    committed trace (identical when parity holds)."""
    import json
    from pathlib import Path

    if golden_npz is not None and Path(golden_npz).exists():
        g = np.load(golden_npz, allow_pickle=False)
        return ([int(x) for x in g["trace_k"]], [int(x) for x in g["trace_locked"]], int(g["lanczos_steps"]),
                f"reference trace ({Path(golden_npz).name})")
    if own_json is not None and Path(own_json).exists():
        d = json.loads(Path(own_json).read_text())
        return ([int(t[2]) for t in d["trace"]], [int(t[1]) for t in d["trace"]], int(d.get("lanczos_steps", 24)),
                f"GPU solve trace ({Path(own_json).name})")
    return None
