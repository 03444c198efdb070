"""Pin the CPU oracle (oracle/bse_oracle.py) to fixtures produced by the
reference package itself (oracle/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden, golden_ham
from oracle import bse_oracle as o


def test_rng_published_words():
    # test_rng.py:6-18 published splitmix64 vectors
    assert o.sm64(0, 0) == 0xE220A8397B1DCDAF
    assert o.sm64(0, 1) == 0x6E789E6AA1B965F4
    assert o.sm64(0xDEADBEEF, 7) == 0xB30A4CCF430B1B5A
    assert o.child_seed(42, 3) == 0x581CE1FF0E4AE394
    z = o.gauss_c(12345, 2)
    assert z[0] == complex(0.56254351858756901, 1.9279936267801181)
    assert z[1] == complex(0.92280219752980885, 1.8429870753916227)


def test_rng_matches_reference_bitwise():
    g = golden("rng.npz")
    assert [o.sm64(0, i) for i in range(16)] == [int(w) for w in g["words_seed0"]]
    assert [o.sm64(0xDEADBEEF, i) for i in range(16)] == [int(w) for w in g["words_deadbeef"]]
    np.testing.assert_array_equal(o.gauss_c(12345, 64), g["normals_12345"])
    np.testing.assert_array_equal(o.gauss_c(o.child_seed(0, 3), 257, first=5), g["normals_sub03"])
    np.testing.assert_array_equal(o.gauss_c_matrix(7, 5, 3), g["matrix_7_5_3"])


def test_generator_matches_reference_small():
    for m, seed in [(8, 11), (16, 5), (32, 4)]:
        a, b = golden_ham(m, seed)
        a2, b2, _ = o.make_instance(m, seed)
        np.testing.assert_allclose(a2, a, rtol=0, atol=1e-12 * np.abs(a).max())
        np.testing.assert_allclose(b2, b, rtol=0, atol=1e-12 * np.abs(b).max())


def test_sub_operators_match_reference():
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    hx = o.h_times(a, b, g["x"])
    np.testing.assert_array_equal(hx, g["hx"])
    fl = [0.0]
    bnd = o.lanczos_bounds(a, b, 6, 16, 2, fl)
    assert bnd.mu_1 == float(g["mu_1"]) and bnd.mu_nevex == float(g["mu_nevex"])
    y = o.cheb_filter(a, b, g["x"], int(g["deg"]), float(g["center"]), float(g["half_width"]),
                      float(g["scale_ref"]))
    np.testing.assert_array_equal(y, g["filtered"])
    q, how = o.cholqr2(y)
    assert how == str(g["method"])
    np.testing.assert_array_equal(q, g["q"])
    lam, vec, lmm = o.rr_hermitian(a, b, q)
    np.testing.assert_allclose(lam, g["rr_values"], rtol=1e-13)
    np.testing.assert_allclose(o.residual_norms(a, b, lam, vec), g["rr_res"], rtol=1e-6, atol=1e-13)
    lam_b, vec_b, _ = o.rr_backup(a, b, q)
    np.testing.assert_allclose(lam_b, g["bk_values"], rtol=1e-12)


@pytest.mark.parametrize("key", ["m64_s21", "m32_s4", "m32_s6", "m32_s8", "m32_s14",
                                 "m48_s12", "m48_s13", "m64_s40", "m24_s100"])
def test_oracle_solve_matches_reference(key):
    import json
    from conftest import GOLDEN
    kw = json.loads((GOLDEN / "meta.json").read_text())["cases"][key]
    m, seed = (int(t[1:]) for t in key.split("_"))
    a, b = golden_ham(m, seed)
    r = o.oracle_solve(a, b, **kw)
    g = golden(f"solve_{key}.npz")
    assert r.iterations_used == int(g["iterations_used"])
    assert r.converged == bool(g["converged"])
    assert r.backup_events == int(g["backup_events"])
    np.testing.assert_allclose(r.lambdas, g["lambdas"], rtol=1e-12, atol=0)
    assert [t["locked"] for t in r.trace] == list(g["trace_locked"])
    assert [t["k"] for t in r.trace] == list(g["trace_k"])
    np.testing.assert_allclose([t["flops"] for t in r.trace], g["trace_flops"], rtol=1e-15)


@pytest.mark.slow
def test_oracle_c1_matches_reference(c1_instance):
    a, b, g = c1_instance
    np.testing.assert_allclose(a @ g["probe"], g["a_probe"], rtol=0, atol=1e-12 * np.abs(g["a_probe"]).max())
    np.testing.assert_array_equal(b[0], g["b_exact_row0"])
    r = o.oracle_solve(a, b, nev=50, nex=20, deg=20, tol=1e-10, seed=0)
    assert r.iterations_used == int(g["abs_iters"]) and r.converged
    assert [t["locked"] for t in r.trace] == list(g["abs_trace_locked"])
    np.testing.assert_allclose(r.lambdas, g["abs_lambdas"], rtol=1e-12)
