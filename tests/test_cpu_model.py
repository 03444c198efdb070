"""The CPU time model of bench.py's reference arm (oracle/cpu_model.py): it times the reference's
code path phase by phase and must reproduce a measured full oracle solve.  Small m here (seconds);
the C2 check on the GPU box's 16 cores is profiles/r02/cpu_model_check_c2.json (model +3.7%)."""
import time

import numpy as np

from oracle import bse_oracle as o
from oracle import cpu_model


def test_phase_model_reproduces_a_measured_solve():
    m, nev, nex = 300, 24, 8
    a, b, _ = o.make_instance(m, 3)
    sec = {}
    t0 = time.perf_counter()
    r = o.oracle_solve(a, b, nev=nev, nex=nex, deg=20, tol=1e-10, rel_res=True, seconds=sec)
    wall = time.perf_counter() - t0
    assert r.converged and set(sec) >= {"lanczos", "filter", "ortho", "rr", "residuals"}
    tk = [t["k"] for t in r.trace]
    tl = [t["locked"] for t in r.trace]
    cal = cpu_model.calibrate(a, b, nev + nex, min(tk), nev)
    mod = cpu_model.model(cal, tk, tl, 20, r.bounds.steps, nevex=nev + nex)
    assert set(mod) == {"lanczos", "filter", "ortho", "rr", "residuals", "start", "total"}
    assert abs(mod["total"] - sum(mod[k] for k in mod if k != "total")) < 1e-9
    # small-m timings are noisy (and this container runs other jobs): a factor-2 sanity band here
    assert 0.5 * wall <= mod["total"] <= 2.0 * wall, (mod, wall, sec)


def test_model_scales_with_the_trace():
    cal = {"k_lo": 100, "k_hi": 1000, "l_hi": 800, "step_100": 1.0, "step_1000": 9.0, "chol_100": 0.1,
           "chol_1000": 5.0, "rr_100": 1.0, "rr_1000": 12.0, "res_100": 1.1, "qr_l": 2.0, "proj_l_khi": 1.0,
           "lanczos_step": 0.1, "start_per_col": 0.001}
    one = cpu_model.model(cal, [1000], [0], 20, 24)
    two = cpu_model.model(cal, [1000, 1000], [10, 20], 20, 24)
    assert two["filter"] == 2 * one["filter"] and two["ortho"] > 2 * one["ortho"]  # the second pays the projection
    np.testing.assert_allclose(one["filter"], 20 * 9.0)
