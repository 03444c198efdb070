"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference golden fixtures.  Tolerances are written next to each check."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_ham
from oracle import bse_oracle as o

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def bse():
    assert torch.cuda.is_available(), "GPU test without a GPU"
    import paper_2601_10557_b200 as m

    return m


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


# ------------------------------------------------------------------ operators
@pytest.mark.parametrize("m,k", [(1, 1), (3, 2), (16, 5), (37, 13), (64, 33), (130, 70), (257, 40), (300, 1), (2001, 1)])
def test_apply_h_matches_oracle(bse, m, k):
    rs = np.random.default_rng(m * 100 + k)
    a0 = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
    a = (a0 + a0.conj().T) / 2
    b0 = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
    b = (b0 + b0.T) / 2
    x = rs.standard_normal((2 * m, k)) + 1j * rs.standard_normal((2 * m, k))
    ham = bse.BseHamiltonian(a, b)
    y = bse.apply_h(ham, x)
    ref = o.h_times(a, b, x)
    assert _rel(y, ref) <= 1e-13  # FP64, different summation order
    ysh = bse.hamiltonian.apply_sh(ham, x)
    assert _rel(ysh, o.s_flip(ref)) <= 1e-13


def test_apply_h_golden(bse):
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    ham = bse.BseHamiltonian(a, b)
    assert _rel(bse.apply_h(ham, g["x"]), g["hx"]) <= 1e-14
    assert _rel(bse.apply_h_via_adjoint(ham, g["x"]), g["hx_adj"]) <= 1e-14
    # 2x2 closed form (test_hamiltonian.py:60-67): H e1 = (2, -0.5)
    h2 = bse.BseHamiltonian(np.array([[2.0]]), np.array([[0.5]]))
    np.testing.assert_allclose(bse.apply_h(h2, np.array([1.0, 0.0])), [2.0, -0.5], atol=1e-15)


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 9), (64, 64, 64), (100, 37, 1000), (33, 129, 4001),
                                   (1200, 1200, 200)])
def test_zgemm_kernels(bse, M, N, K):
    from paper_2601_10557_b200 import _lib
    from paper_2601_10557_b200.hamiltonian import to_colmajor, colmajor_empty, ld_of

    rs = np.random.default_rng(M + N + K)
    ctx = _lib.Context.get(0)
    dev = torch.device("cuda", 0)
    a = rs.standard_normal((K, M)) + 1j * rs.standard_normal((K, M))
    b = rs.standard_normal((K, N)) + 1j * rs.standard_normal((K, N))
    c0 = rs.standard_normal((M, N)) + 1j * rs.standard_normal((M, N))
    da, db, dc = to_colmajor(a, dev), to_colmajor(b, dev), to_colmajor(c0, dev)
    ctx.call("bse_zgemm_cn", M, N, K, 2.0, _lib.dptr(da), ld_of(da), _lib.dptr(db), ld_of(db), 0.5, _lib.dptr(dc),
             ld_of(dc))
    got = dc.T.contiguous().cpu().numpy().T
    assert _rel(got, 2.0 * a.conj().T @ b + 0.5 * c0) <= 1e-13
    an = rs.standard_normal((M, K)) + 1j * rs.standard_normal((M, K))
    dan = to_colmajor(an, dev)
    dc2 = colmajor_empty(M, N, dev)
    ctx.call("bse_zgemm_nn", M, N, K, -1.0, _lib.dptr(dan), ld_of(dan), _lib.dptr(db), ld_of(db), 0.0, _lib.dptr(dc2),
             ld_of(dc2))
    assert _rel(dc2.T.contiguous().cpu().numpy().T, -(an @ b)) <= 1e-13


def test_filter_golden(bse):
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    ham = bse.BseHamiltonian(a, b)
    cfg = bse.FilterConfig(int(g["deg"]), float(g["center"]), float(g["half_width"]), float(g["scale_ref"]))
    out = bse.chebyshev_filter(ham, g["x"], cfg)
    assert _rel(out, g["filtered"]) <= 1e-12  # test_chebyshev.py:110-117 uses 1e-12 x scale


def test_filter_scalar_consistency_on_eigenpairs(bse):
    # test_chebyshev.py:54-61: filter on every eigenvector equals the scalar gain
    a, b = golden_ham(8, 11)
    ham = bse.BseHamiltonian(a, b)
    h = o.dense_h(a, b)
    lam, vecs = np.linalg.eig(h)
    order = np.argsort(lam.real)
    lam, vecs = lam.real[order], vecs[:, order]
    bnd = bse.estimate_bounds(ham, nevex=4, steps=16, seed=2)
    cfg = bse.FilterConfig.from_bounds(bnd, 12)
    out = bse.chebyshev_filter(ham, vecs, cfg)
    for i in range(lam.shape[0]):
        gain = bse.scalar_filter_value(lam[i], cfg)
        assert np.linalg.norm(out[:, i] - gain * vecs[:, i]) <= 1e-10 * max(abs(gain), 1.0)


def test_lanczos_bounds_golden(bse):
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    bnd = bse.estimate_bounds(bse.BseHamiltonian(a, b), nevex=6, steps=16, seed=2)
    assert bnd.steps == int(g["steps"])
    assert abs(bnd.mu_1 - float(g["mu_1"])) <= 1e-12 * abs(float(g["mu_1"]))
    assert abs(bnd.mu_nevex - float(g["mu_nevex"])) <= 1e-10 * abs(float(g["mu_1"]))


def test_cholqr_matches_oracle(bse):
    g = golden("ops_m16_s5.npz")
    q, method = bse.cholqr_with_fallback(g["filtered"])
    assert method == "cholqr"
    assert np.abs(q.conj().T @ q - np.eye(q.shape[1])).max() <= 1e-12
    # phase-fixed Q is unique: compare with the reference's Q (cond-limited)
    assert _rel(q, g["q"]) <= 1e-8


def _rand(n, k, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal((n, k)) + 1j * g.standard_normal((n, k))


def test_cholqr_fallback_and_rank(bse):
    # test_ortho.py:22-28, 43-53: singular values clustered at 1 and 1e-8 force the
    # fallback (shifted CholQR3 here, Householder in the reference); v, v + 1e-12 w is
    # numerically rank deficient; k > n is rejected
    u, _ = np.linalg.qr(_rand(60, 6, 0))
    v, _ = np.linalg.qr(_rand(6, 6, 1))
    s = np.ones(6)
    s[3:] = 1e-8
    x = u @ np.diag(s) @ v.conj().T
    q, method = bse.cholqr_with_fallback(x)
    assert method == "shifted_cholqr"
    assert np.abs(q.conj().T @ q - np.eye(6)).max() <= 1e-12
    vv, ww = _rand(30, 1, 4), _rand(30, 1, 5)
    with pytest.raises(bse.RankDeficiencyError):
        bse.cholqr_with_fallback(np.concatenate([vv, vv + 1e-12 * ww], axis=1))
    with pytest.raises(bse.RankDeficiencyError):
        bse.cholqr_with_fallback(_rand(3, 5, 6))
    q, method = bse.cholqr_with_fallback(np.eye(6, 3, dtype=complex))
    assert method == "cholqr" and np.abs(q - np.eye(6, 3)).max() <= 1e-14
    q, _ = bse.cholqr_with_fallback(_rand(20, 4, 7))
    for j in range(4):  # phase convention test_ortho.py:61-66
        lead = np.nonzero(np.abs(q[:, j]) >= 1e-8 * np.abs(q[:, j]).max())[0][0]
        assert abs(q[lead, j].imag) <= 1e-14 and q[lead, j].real > 0


def test_s_orthonormalize_against_locked(bse):
    a, b = golden_ham(32, 4)
    rs = np.random.default_rng(1)
    y = rs.standard_normal((64, 3)) + 1j * rs.standard_normal((64, 3))
    y /= np.linalg.norm(y, axis=0)
    v = rs.standard_normal((64, 5)) + 1j * rs.standard_normal((64, 5))
    space, method = bse.s_orthonormalize(v, y)
    qa = space.active
    assert space.locked == 3 and np.array_equal(space.locked_cols, y)
    assert np.abs((o.s_flip(y)).conj().T @ qa).max() <= 1e-10  # test_ortho.py:82-103
    assert np.abs(qa.conj().T @ qa - np.eye(5)).max() <= 1e-12
    ref, _ = o.s_ortho(v, y)
    # same subspace: singular values of ref^H qa all 1
    sv = np.linalg.svd(ref.conj().T @ qa, compute_uv=False)
    assert np.abs(sv - 1).max() <= 1e-10


def test_rayleigh_ritz_golden(bse):
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    ham = bse.BseHamiltonian(a, b)
    ritz, red = bse.build_hermitian_rq(ham, g["q"])
    assert np.abs(ritz.values - g["rr_values"]).max() <= 1e-12 * np.abs(g["rr_values"]).max()
    assert abs(red.lambda_min_m - float(g["rr_lambda_min_m"])) <= 1e-12
    res = bse.residuals(ham, ritz)
    np.testing.assert_allclose(res, g["rr_res"], rtol=1e-6, atol=1e-12)
    # Ritz vectors: phase-invariant agreement per column
    ov = np.abs(np.einsum("ij,ij->j", ritz.vectors.conj(), g["rr_vectors"]))
    assert np.abs(ov - 1).max() <= 1e-10
    rb, redb = bse.build_backup_rq(ham, g["q"])
    assert np.abs(rb.values - g["bk_values"]).max() <= 1e-10 * np.abs(g["bk_values"]).max()
    # the reduced problems as the reference returns them (rayleigh_ritz.py:41-51, 140-143, 176-179)
    sc = np.abs(g["rr_w"]).max()
    assert red.variant == "hermitian" and red.d is None
    assert _rel(red.w, g["rr_w"]) <= 1e-12 and _rel(red.m, g["rr_m"]) <= 1e-12 and _rel(red.g, g["rr_g"]) <= 1e-11
    assert np.allclose(np.triu(red.l, 1), 0) and np.abs(red.l @ red.l.conj().T - red.w).max() <= 1e-12 * sc
    assert redb.variant == "backup" and redb.l is None and redb.d.shape == (g["q"].shape[1],)
    np.testing.assert_allclose(redb.d, np.real(np.diag(red.m)), rtol=0, atol=1e-14)
    assert _rel(redb.m, g["rr_m"]) <= 1e-12
    # backup G = diag(d)^-1 (Q^H S H Q - offdiag(M) Q^H H Q): its eigenvalues are the backup Ritz values
    assert np.abs(np.sort(np.linalg.eigvals(redb.g).real) - g["bk_values"]).max() <= 1e-9 * np.abs(g["bk_values"]).max()


def test_rr_products_on_real_split_planes(bse):
    """The RR's T = S H Q (hermitian) and T = H Q (backup) on the registered real-split planes
    (bse_set_rs_planes, csrc/hop_rs.cuh) against the 3M products: Ritz values within 1e-12, Ritz
    vectors phase-invariantly within 1e-10, the registration scoped to the call."""
    a, b = golden_ham(64, 21)
    rng = np.random.default_rng(2)
    q, _ = np.linalg.qr(rng.standard_normal((128, 24)) + 1j * rng.standard_normal((128, 24)))
    default = bse.filter_algorithm()
    out = {}
    try:
        for algo in ("3m", "rs"):
            bse.set_filter_algorithm(algo)
            ham = bse.BseHamiltonian(a, b)
            ritz, _ = bse.build_hermitian_rq(ham, q)
            rb, _ = bse.build_backup_rq(ham, q)
            out[algo] = (ritz, rb, ham)
    finally:
        bse.set_filter_algorithm(default)
    (r3, b3, _), (rr, br, ham_rs) = out["3m"], out["rs"]
    assert ham_rs.device_rs_planes(0) is not None
    scale = np.abs(r3.values).max()
    assert np.abs(rr.values - r3.values).max() <= 1e-12 * scale
    assert np.abs(br.values - b3.values).max() <= 1e-12 * scale
    ov = np.abs(np.einsum("ij,ij->j", np.asarray(rr.vectors).conj(), np.asarray(r3.vectors)))
    assert np.abs(ov - 1).max() <= 1e-10


def test_rr_exact_invariant_subspace(bse):
    # test_rayleigh_ritz.py:48-58: RR on an exact invariant subspace reproduces eigenpairs
    a, b = golden_ham(8, 11)
    lam = o.dense_eigs(a, b)
    h = o.dense_h(a, b)
    w, vecs = np.linalg.eig(h)
    idx = np.argsort(w.real)[:4]
    q, _ = np.linalg.qr(vecs[:, idx])
    ritz, _ = bse.build_hermitian_rq(bse.BseHamiltonian(a, b), q)
    assert np.abs(ritz.values - lam[:4]).max() <= 1e-10 * np.abs(lam).max()


# ------------------------------------------------------------------ generator
@pytest.mark.parametrize("m,seed", [(8, 11), (16, 5), (32, 4), (64, 21)])
def test_generator_matches_reference(bse, m, seed):
    a, b = golden_ham(m, seed)
    ham = bse.generate(bse.GeneratorSpec(m=m, seed=seed))
    ga, gb = ham.host_blocks()
    assert _rel(ga, a) <= 1e-14
    assert _rel(gb, b) <= 1e-13
    assert ham.definiteness is bse.Definiteness.DEFINITE


def test_generator_device_rng_close_to_host(bse):
    hx = bse.generate(bse.GeneratorSpec(m=40, seed=3), exact=True)
    hd = bse.generate(bse.GeneratorSpec(m=40, seed=3), exact=False)
    ax, _ = hx.host_blocks()
    ad, _ = hd.host_blocks()
    assert _rel(ad, ax) <= 1e-13  # words bit-exact, device libm within ulps


# ------------------------------------------------------------------ full solves
@pytest.mark.parametrize("key", ["m64_s21", "m32_s4", "m32_s6", "m32_s8", "m32_s14", "m48_s12", "m48_s13",
                                 "m64_s40", "m24_s100"])
def test_solve_matches_reference(bse, key):
    kw = json.loads((GOLDEN / "meta.json").read_text())["cases"][key]
    m, seed = (int(t[1:]) for t in key.split("_"))
    a, b = golden_ham(m, seed)
    res = bse.solve(bse.BseHamiltonian(a, b), bse.SolverConfig(**kw))
    g = golden(f"solve_{key}.npz")
    assert res.converged == bool(g["converged"])
    assert abs(res.iterations_used - int(g["iterations_used"])) <= 1  # north star: +-1 outer iteration
    if res.iterations_used == int(g["iterations_used"]):
        assert [t.locked for t in res.trace] == list(g["trace_locked"])
        assert [t.k for t in res.trace] == list(g["trace_k"])
        np.testing.assert_allclose([t.flops for t in res.trace], g["trace_flops"], rtol=1e-15)
    rel = np.abs(res.lambdas - g["lambdas"]) / np.abs(g["lambdas"])
    assert rel.max() <= (1e-10 if res.converged else 1e-6)  # 1e-10 relative in complex128
    tol = kw.get("tol", 1e-8) * (abs(res.bounds.mu_1) if kw.get("rel_res") else 1.0)
    if res.converged:
        assert res.residual_norms.max() <= tol
    # phase-invariant subspace check (|v_ref^H v| = 1 per simple pair)
    ov = np.abs(np.einsum("ij,ij->j", g["v"].conj(), res.v))
    if res.converged:
        assert np.abs(ov - 1).max() <= 1e-8


def test_solve_2x2_and_tda(bse):
    lam2 = np.sqrt(3.75)
    ham = bse.BseHamiltonian(np.diag([2.0, 2.0]), np.diag([0.5, 0.5]))
    r = bse.solve(ham, bse.SolverConfig(nev=1, nex=1, lanczos_steps=2, seed=3))
    assert r.converged and abs(r.lambdas[0] + lam2) <= 1e-10
    a = np.diag(np.arange(1.0, 9.0))
    r = bse.solve(bse.BseHamiltonian(a, np.zeros((8, 8))), bse.SolverConfig(nev=3, nex=3, deg=8, lanczos_steps=4, seed=1))
    assert r.converged
    np.testing.assert_allclose(r.lambdas, [-8.0, -7.0, -6.0], atol=1e-8)
    assert np.abs(r.v[:8]).max() <= 1e-6


def test_solve_errors(bse):
    ham = bse.BseHamiltonian(np.array([[1.0]]), np.array([[2.0]]))
    with pytest.raises(bse.IndefiniteError):
        bse.solve(ham, bse.SolverConfig(nev=1, nex=0, deg=2, lanczos_steps=2))
    a, b = golden_ham(8, 11)
    with pytest.raises(bse.ValidationError):
        bse.solve(bse.BseHamiltonian(a, b), bse.SolverConfig(nev=5, nex=5))


def test_solve_deterministic(bse):
    a, b = golden_ham(32, 4)
    ham = bse.BseHamiltonian(a, b)
    r1 = bse.solve(ham, bse.SolverConfig(nev=4, seed=9))
    r2 = bse.solve(ham, bse.SolverConfig(nev=4, seed=9))
    np.testing.assert_array_equal(r1.lambdas, r2.lambdas)
    np.testing.assert_array_equal(r1.v, r2.v)


def test_c1_parity(bse, c1_instance):
    """BASELINE configs[0]: m=500 (n=1000), nev=50, nex=20, deg=20, abs tol 1e-10 and rel_res."""
    a, b, g = c1_instance
    ham = bse.BseHamiltonian(a, b)
    for tag, rel_res in (("abs", False), ("rel", True)):
        r = bse.solve(ham, bse.SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0, rel_res=rel_res))
        assert r.converged
        assert abs(r.iterations_used - int(g[f"{tag}_iters"])) <= 1
        rel = np.abs(r.lambdas - g[f"{tag}_lambdas"]) / np.abs(g[f"{tag}_lambdas"])
        assert rel.max() <= 1e-10
        thr = 1e-10 * (abs(r.bounds.mu_1) if rel_res else 1.0)
        assert r.residual_norms.max() <= thr
        ov = np.abs(np.einsum("ij,ij->j", g[f"{tag}_v10"].conj(), r.v[:, :10]))
        assert np.abs(ov - 1).max() <= 1e-8


@pytest.mark.parametrize("algo", ["3m", "3m-tma-narrow", "3m-tma-wide", "4m", "rs", "rs-tall4-k32", "rs-tall4", "rs-tall", "rs-narrow"])
def test_filter_3m_accuracy_and_c1_parity(bse, c1_instance, algo):
    """3M (Gauss) filter products: the filter output within 1e-12 of the 4M result (scaled), and
    the C1 solve (abs tol 1e-10) keeps the reference's iterations +-1 and lambda to 1e-10 relative."""
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    ham = bse.BseHamiltonian(a, b)
    cfg = bse.FilterConfig(int(g["deg"]), float(g["center"]), float(g["half_width"]), float(g["scale_ref"]))
    default = bse.filter_algorithm()
    try:
        bse.set_filter_algorithm(algo)
        out3 = bse.chebyshev_filter(ham, g["x"], cfg)
        a1, b1, gc = c1_instance
        r = bse.solve(bse.BseHamiltonian(a1, b1), bse.SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0))
    finally:
        bse.set_filter_algorithm(default)
    assert _rel(out3, g["filtered"]) <= 1e-12
    assert r.converged and abs(r.iterations_used - int(gc["abs_iters"])) <= 1
    assert (np.abs(r.lambdas - gc["abs_lambdas"]) / np.abs(gc["abs_lambdas"])).max() <= 1e-10
    assert r.residual_norms.max() <= 1e-10


def test_filter_3m_variants_bitwise_identical(bse):
    """Every 3M kernel variant (barrier / mbarrier / TMA feeds, all tile shapes, the k-dispatched
    default) accumulates each output in the same K order: identical bits at ragged shapes."""
    import torch
    from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of
    from paper_2601_10557_b200 import _lib

    dev = torch.device("cuda", 0)
    ctx = _lib.Context.get(0)
    m, k, deg = 203, 530, 4  # ragged in rows, K and columns; k >= 512 takes the wide default tile
    gen = torch.Generator(device=dev).manual_seed(5)
    ab = colmajor_empty(m, 2 * m, dev)
    ab.copy_(torch.complex(torch.randn(m, 2 * m, generator=gen, device=dev, dtype=torch.float64),
                           torch.randn(m, 2 * m, generator=gen, device=dev, dtype=torch.float64)))
    sd = colmajor_empty(m, 2 * m, dev)
    ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m, _lib.dptr(sd))
    v0 = colmajor_empty(2 * m, k, dev)
    v0.copy_(torch.complex(torch.randn(2 * m, k, generator=gen, device=dev, dtype=torch.float64),
                           torch.randn(2 * m, k, generator=gen, device=dev, dtype=torch.float64)))
    work = torch.empty(2 * 2 * m * k, dtype=torch.complex128, device=dev)
    outs = {}
    default = bse.filter_algorithm()
    try:
        for algo in ("3m", "3m-tma-narrow", "3m-tma-wide"):
            bse.set_filter_algorithm(algo)
            for kk in (k, 100):  # both sides of the default's column threshold
                v = v0[:, :kk].clone()
                v = v.T.contiguous().T
                ctx.call("bse_chebyshev_filter", _lib.dptr(ab), _lib.dptr(sd), ld_of(ab), m, _lib.dptr(v), 2 * m, kk,
                         deg, 0.5, 2.0, -3.0, _lib.dptr(work))
                outs[(algo, kk)] = v.cpu()
    finally:
        bse.set_filter_algorithm(default)
    for (algo, kk), v in outs.items():
        assert torch.equal(v, outs[("3m", kk)]), (algo, kk)


@pytest.mark.parametrize("ksplit", [2, 3, 4])
def test_rs_split_k(ksplit):
    """Split-K real-split products (hop_rs.cuh: a tile's contraction over ksplit CTAs, partial sums
    reduced in fixed order by rs_splitk_epilogue_kernel): filter and transposed-tile product within
    rounding of the unsplit tile, deterministic run to run; ragged shapes including splits left
    without K stages (kc = 5 over 3 or 4 CTAs)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, BSE200_RS_KSPLIT=str(ksplit))
    worker = Path(__file__).resolve().parent / "_splitk_worker.py"
    r = subprocess.run([sys.executable, str(worker)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(rows) == 4
    for row in rows:
        assert row["filter_rel"] <= 1e-13 and row["trans_rel"] <= 1e-14, row
        assert row["repeat_bitwise"], row


def test_filter_rs_matches_3m_and_tiles_bitwise(bse):
    """Real-split filter (csrc/hop_rs.cuh: folded basis, four real planes, 4 n^2 k flops per step)
    against the 3M filter at ragged shapes: within 1e-12 of the output scale; its tile variants
    accumulate each output in the same K order, so they agree bit for bit."""
    import torch
    from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of
    from paper_2601_10557_b200 import _lib

    dev = torch.device("cuda", 0)
    ctx = _lib.Context.get(0)
    gen = torch.Generator(device=dev).manual_seed(9)
    default = bse.filter_algorithm()
    try:
        for m, k in ((203, 530), (203, 100), (37, 7), (1, 1)):
            ab = colmajor_empty(m, 2 * m, dev)
            ab.copy_(torch.complex(torch.randn(m, 2 * m, generator=gen, device=dev, dtype=torch.float64),
                                   torch.randn(m, 2 * m, generator=gen, device=dev, dtype=torch.float64)))
            sd = colmajor_empty(m, 2 * m, dev)
            ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m, _lib.dptr(sd))
            ldg = m + (m & 1)
            gp = torch.empty((4 * m, ldg), dtype=torch.float64, device=dev).t()
            ctx.call("bse_make_rs_planes", _lib.dptr(ab), ld_of(ab), m, m, _lib.dptr(gp), ldg)
            v0 = colmajor_empty(2 * m, k, dev)
            v0.copy_(torch.complex(torch.randn(2 * m, k, generator=gen, device=dev, dtype=torch.float64),
                                   torch.randn(2 * m, k, generator=gen, device=dev, dtype=torch.float64)))
            work = torch.empty(2 * 2 * m * k, dtype=torch.complex128, device=dev)
            bse.set_filter_algorithm("3m")
            ref = v0.clone()
            ctx.call("bse_chebyshev_filter", _lib.dptr(ab), _lib.dptr(sd), ld_of(ab), m, _lib.dptr(ref), 2 * m, k, 4,
                     0.5, 2.0, -3.0, _lib.dptr(work))
            outs = {}
            for algo in ("rs", "rs-tall4-k32", "rs-tall4", "rs-tall", "rs-narrow"):
                bse.set_filter_algorithm(algo)
                v = v0.clone()
                ctx.call("bse_chebyshev_filter_rs", _lib.dptr(gp), ldg, m, _lib.dptr(v), 2 * m, k, 4, 0.5, 2.0, -3.0,
                         _lib.dptr(work))
                outs[algo] = v
            scale = ref.abs().max().item()
            assert (outs["rs"] - ref).abs().max().item() <= 1e-12 * scale, (m, k)
            for algo, v in outs.items():
                assert torch.equal(v, outs["rs"]), (algo, m, k)
    finally:
        bse.set_filter_algorithm(default)


def test_fused_residuals_match_explicit(bse, c1_instance):
    """(H Q) w residuals vs the explicit H (Q w) product of rayleigh_ritz.py:188."""
    from paper_2601_10557_b200.hamiltonian import to_colmajor
    from paper_2601_10557_b200.rayleigh_ritz import build_hermitian_rq_device, residuals_device

    a, b, _ = c1_instance
    ham = bse.BseHamiltonian(a, b)
    g = golden("ops_m16_s5.npz")
    rs = np.random.default_rng(0)
    for h, q in ((bse.BseHamiltonian(*golden_ham(16, 5)), g["q"]),
                 (ham, np.linalg.qr(rs.standard_normal((1000, 40)) + 1j * rs.standard_normal((1000, 40)))[0])):
        qd = to_colmajor(q, torch.device("cuda", 0))
        r, _ = build_hermitian_rq_device(h, qd, fused_residuals=True)
        explicit = residuals_device(h, r.values, r.vectors)
        scale = np.abs(r.values).max()
        assert np.all(np.abs(r.residual_norms - explicit) <= 1e-12 * scale + 1e-10 * explicit)
    # a full C1 solve under the relative policy with fused residuals keeps parity
    r = bse.solve(ham, bse.SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0, rel_res=True))
    gc = c1_instance[2]
    assert r.converged and abs(r.iterations_used - int(gc["rel_iters"])) <= 1
    assert (np.abs(r.lambdas - gc["rel_lambdas"]) / np.abs(gc["rel_lambdas"])).max() <= 1e-10


def test_pchb_device_reader_and_cli_solve(bse, tmp_path):
    from paper_2601_10557_b200 import fileio
    from paper_2601_10557_b200.cli import main

    hd = fileio.read_pchb(GOLDEN / "m8_s11.pchb", device=torch.device("cuda", 0))
    a, b = golden_ham(8, 11)
    ga, gb = hd.host_blocks()
    np.testing.assert_array_equal(ga, a)
    np.testing.assert_array_equal(gb, b)
    rc = main(["solve", "--pchb", str(GOLDEN / "m8_s11.pchb"), "--nev", "2", "--tol", "1e-10", "--out", str(tmp_path)])
    assert rc == 0
    lines = (tmp_path / "eigenvalues.csv").read_text().splitlines()
    assert lines[0] == "# bsesolve eigenvalues v1" and lines[4] == "index,eigenvalue,residual" and len(lines) == 7
    lam = np.array([float(l.split(",")[1]) for l in lines[5:]])
    ref = o.dense_eigs(a, b)[:2]
    assert np.abs(lam - ref).max() <= 1e-10 * np.abs(ref).max()
    v = fileio.read_pchv(tmp_path / "eigenvectors.bin")
    assert v.shape == (16, 2)
    assert (tmp_path / "trace.csv").exists() and (tmp_path / "manifest.json").exists()


@pytest.mark.parametrize("pair", ["0", "1"])
def test_c64_tcgen05_filter_accuracy(bse, monkeypatch, pair):
    """complex64 filter on tcgen05 (3xTF32): the filter output within FP32 accuracy of the
    reference's complex128 filter (golden), and of the oracle on a ragged shape; with the
    single-CTA kernel and the CTA-pair (cta_group::2) kernel (m = 300: 3 row tiles, so the
    last pair holds an all-padding CTA)."""
    monkeypatch.setenv("BSE200_C64_PAIR", pair)
    a, b = golden_ham(16, 5)
    g = golden("ops_m16_s5.npz")
    ham = bse.BseHamiltonian(a, b)
    cfg = bse.FilterConfig(int(g["deg"]), float(g["center"]), float(g["half_width"]), float(g["scale_ref"]))
    try:
        bse.set_filter_precision("c64")
        out = bse.chebyshev_filter(ham, g["x"], cfg)
        rs = np.random.default_rng(7)
        m = 300
        a2 = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
        a2 = a2 @ a2.conj().T / m + np.eye(m)
        b2 = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
        b2 = 0.1 * (b2 + b2.T) / 2
        x2 = rs.standard_normal((2 * m, 130)) + 1j * rs.standard_normal((2 * m, 130))
        h2 = bse.BseHamiltonian(a2, b2)
        c2 = bse.FilterConfig(6, 1.0, 3.0, -5.0)
        out2 = bse.chebyshev_filter(h2, x2, c2)
    finally:
        bse.set_filter_precision("c128")
    assert _rel(out, g["filtered"]) <= 2e-5  # FP32 arithmetic (3xTF32 products, fp32 accumulation)
    ref2 = o.cheb_filter(a2, b2, x2, 6, 1.0, 3.0, -5.0)
    assert _rel(out2, ref2) <= 2e-5


def test_c64_solve_c1_parity(bse, c1_instance):
    """C1 with the complex64 filter under the c64 policy (rel_res, tol 1e-5):
    eigenvalues within 1e-4 relative of the complex128 reference."""
    a, b, g = c1_instance
    try:
        bse.set_filter_precision("c64")
        r = bse.solve(bse.BseHamiltonian(a, b), bse.SolverConfig(nev=50, nex=20, deg=20, tol=1e-5, seed=0,
                                                                  rel_res=True))
    finally:
        bse.set_filter_precision("c128")
    assert r.converged
    rel = np.abs(r.lambdas - g["rel_lambdas"]) / np.abs(g["rel_lambdas"])
    assert rel.max() <= 1e-4
    assert r.residual_norms.max() <= 1e-5 * abs(r.bounds.mu_1)


def test_mixed_precision_solve_parity(bse, c1_instance, monkeypatch):
    """Mixed-precision ChASE (early filters complex64 on tcgen05, later FP64): C1 under both
    tolerance policies keeps the reference's eigenvalues (1e-10 rel), residuals and iterations +-1."""
    monkeypatch.setenv("BSE200_MIXED", "1")
    a, b, g = c1_instance
    ham = bse.BseHamiltonian(a, b)
    for tag, rel in (("abs", False), ("rel", True)):
        r = bse.solve(ham, bse.SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0, rel_res=rel))
        assert r.converged and "c64" in r.filter_precisions and r.filter_precisions[-1] == "c128"
        assert abs(r.iterations_used - int(g[f"{tag}_iters"])) <= 1
        assert (np.abs(r.lambdas - g[f"{tag}_lambdas"]) / np.abs(g[f"{tag}_lambdas"])).max() <= 1e-10
        assert r.residual_norms.max() <= 1e-10 * (abs(r.bounds.mu_1) if rel else 1.0)


def test_abi_validation_errors(bse):
    """Status codes of the entry points added for the grid and kernel selection map onto the
    reference exception classes (errors.py:8-38) and fire before any device work."""
    import ctypes

    from paper_2601_10557_b200 import _lib

    ctx = _lib.Context.get(0)
    with pytest.raises(bse.ValidationError):
        ctx.call("bse_set_filter_algorithm", 99)
    with pytest.raises(bse.ValidationError):
        ctx.call("bse_rr_pencil_part", 3, None, None, 4, None, None, None)
    args = _lib.C64TileArgs()
    args.mo, args.kc, args.k = 8, 0, 4
    with pytest.raises(bse.ValidationError):
        ctx.call("bse_c64_tile_step", ctypes.byref(args))
    with pytest.raises(bse.ValidationError):
        ctx.call("bse_c64_tile_planes", None, None, 2, 8, 4, None)  # lds < kc
    ctx.call("bse_set_filter_algorithm", _lib._ALGOS[bse.filter_algorithm()])  # context stays usable


def test_filter_without_sum_planes_when_hbm_is_short(bse, monkeypatch):
    """When the 3M sum planes (+32 m^2 bytes) would not fit next to the solve (n = 100k on one GPU),
    the filter and the RR product form the operand sums in registers instead: same 3M arithmetic,
    same results."""
    from paper_2601_10557_b200 import _lib
    from paper_2601_10557_b200.dist import DistributedSolver

    a, b = golden_ham(64, 21)
    cfg = bse.FilterConfig(10, 300.0, 250.0, -600.0)
    x = np.random.default_rng(3).standard_normal((128, 40)) + 1j * np.random.default_rng(4).standard_normal((128, 40))
    with_planes = bse.chebyshev_filter(bse.BseHamiltonian(a, b), x, cfg)
    monkeypatch.setattr(_lib, "planes_fit", lambda *args, **kw: False)
    ham = bse.BseHamiltonian(a, b)
    without = bse.chebyshev_filter(ham, x, cfg)
    assert ham.device_sum_planes(0) is None
    assert _rel(without, with_planes) <= 1e-13
    r = bse.solve(bse.BseHamiltonian(a, b), bse.SolverConfig(nev=8, seed=21))
    g = golden("solve_m64_s21.npz")
    assert (np.abs(r.lambdas - g["lambdas"]) / np.abs(g["lambdas"])).max() <= 1e-10
    ds = DistributedSolver((a, b))
    rd = ds.solve(bse.SolverConfig(nev=8, seed=21))
    assert ds.fwd.sd is None and (np.abs(rd.lambdas - g["lambdas"]) / np.abs(g["lambdas"])).max() <= 1e-10


def test_complete_spectrum_and_mirror_largest_match_reference(bse):
    """solver.py:253-299 on the drop-in's own solve, against the reference's outputs for its solve
    of the same case (tests/golden/post_m32_s4.npz, oracle/make_golden_post.py): values exactly
    as ordered, vectors per column up to a phase (the Ritz vectors' phase is the eigensolver's)."""
    a, b = golden_ham(32, 4)
    g = golden("post_m32_s4.npz")
    r = bse.solve(bse.BseHamiltonian(a, b), bse.SolverConfig(nev=4, seed=9))
    assert np.abs(r.lambdas - g["lambdas"]).max() <= 1e-10 * np.abs(g["lambdas"]).max()

    def same_up_to_phase(x, y):
        ov = np.abs(np.einsum("ij,ij->j", x.conj(), y)) / (np.linalg.norm(x, axis=0) * np.linalg.norm(y, axis=0))
        return np.abs(ov - 1).max()

    cs = bse.complete_spectrum(r)
    assert np.abs(cs.values - g["cs_values"]).max() <= 1e-10 * np.abs(g["cs_values"]).max()
    assert same_up_to_phase(cs.right, g["cs_right"]) <= 1e-10
    assert same_up_to_phase(cs.left, g["cs_left"]) <= 1e-10
    # left pairs: u_i^H v_j = 0 for i != j and the sign normalisation u^H v > 0 (solver.py:262-266)
    d = cs.left.conj().T @ cs.right
    assert np.abs(d - np.diag(np.diag(d))).max() <= 1e-8 and (np.real(np.diag(d)) > 0).all()
    ml = bse.mirror_largest(r)
    assert np.abs(ml.lambdas - g["ml_lambdas"]).max() <= 1e-10 * np.abs(g["ml_lambdas"]).max()
    assert same_up_to_phase(ml.v, g["ml_v"]) <= 1e-10
    np.testing.assert_allclose(ml.residual_norms, r.residual_norms[np.argsort(-r.lambdas, kind="stable")])


def test_cli_bench_matches_reference_format(bse, tmp_path):
    """`bench` subcommand (cli.py:291-361): bench.csv with the reference's header, input digest,
    (rep, phase) rows and modeled flops -- identical to the reference's own bench.csv on the same
    PCHB (tests/golden/m8_s11_bench.csv) except the measured seconds -- plus manifest.json."""
    from paper_2601_10557_b200.cli import main

    rc = main(["bench", "--pchb", str(GOLDEN / "m8_s11.pchb"), "--nev", "2", "--tol", "1e-10", "--reps", "2",
               "--out", str(tmp_path)])
    assert rc == 0
    got = (tmp_path / "bench.csv").read_text().splitlines()
    ref = (GOLDEN / "m8_s11_bench.csv").read_text().splitlines()
    assert got[:4] == ref[:4] and len(got) == len(ref)
    for gl, rl in zip(got[4:], ref[4:]):
        gf, rf = gl.split(","), rl.split(",")
        assert gf[:2] == rf[:2] and gf[3] == rf[3], (gl, rl)  # rep, phase, modeled flops
    assert json.loads((tmp_path / "manifest.json").read_text())["command"] == "bench"


def test_planes_only_operator_solve(bse):
    """The operator held as its real-split planes only (drop_blocks_for_planes: n = 100k on one GPU,
    where [A|B] and the planes do not both fit): Lanczos (k = 1 matvecs), filter, RR and fused
    residuals all on the planes; same results as with [A|B] kept, and A, B recoverable from the
    planes to rounding."""
    import torch

    a, b = golden_ham(64, 21)
    g = golden("solve_m64_s21.npz")
    ham = bse.BseHamiltonian(a, b)
    dev = torch.device("cuda", 0)
    ham.device_blocks(dev)
    assert ham.drop_blocks_for_planes(dev) and ham.planes_only(dev) and ham.device_blocks(dev) is None
    r = bse.solve(ham, bse.SolverConfig(nev=8, seed=21, rel_res=True, tol=1e-12))
    ref = bse.solve(bse.BseHamiltonian(a, b), bse.SolverConfig(nev=8, seed=21, rel_res=True, tol=1e-12))
    assert r.iterations_used == ref.iterations_used
    assert [t.locked for t in r.trace] == [t.locked for t in ref.trace]
    assert np.abs(r.lambdas - ref.lambdas).max() <= 1e-12 * np.abs(ref.lambdas).max()
    assert np.abs(r.lambdas - g["dense_lambdas"][:8]).max() <= 1e-10 * np.abs(g["dense_lambdas"][:8]).max()
    born = bse.generate(bse.GeneratorSpec(m=64, seed=21))  # device-born: A, B come back from the planes
    ga, gb = born.host_blocks()
    born2 = bse.generate(bse.GeneratorSpec(m=64, seed=21))
    assert born2.drop_blocks_for_planes(dev)
    ra, rb = born2.host_blocks()
    # each plane entry is one rounded add of A and B entries: errors of order eps |A| in both blocks
    scale = np.abs(ga).max()
    assert np.abs(ra - ga).max() <= 4e-16 * scale and np.abs(rb - gb).max() <= 4e-16 * scale


def test_split_start_block_and_first_filter_change_no_bit(bse, monkeypatch):
    """The start block drawn in two column halves with the first filter run per half (solver.py;
    the host draws the second half while the GPU filters the first) gives bitwise the same solve
    (at sizes where the real-split products of both widths take the same split-K plan, as here)."""
    import paper_2601_10557_b200.solver as solver_mod

    a, b = golden_ham(64, 21)
    cfg = bse.SolverConfig(nev=8, seed=21)
    monkeypatch.setattr(solver_mod, "START_SPLIT_MIN", 1 << 30)
    whole = bse.solve(bse.BseHamiltonian(a, b), cfg)
    monkeypatch.setattr(solver_mod, "START_SPLIT_MIN", 4)
    split = bse.solve(bse.BseHamiltonian(a, b), cfg)
    assert np.array_equal(whole.lambdas, split.lambdas) and np.array_equal(whole.v, split.v)
    assert [t.locked for t in whole.trace] == [t.locked for t in split.trace]
