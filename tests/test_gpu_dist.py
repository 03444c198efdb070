"""GPU checks of the 2D-distributed code path (paper_2601_10557_b200/dist.py) with the
CUDA ops: world size 1 in-process here; N = 2 / 4 through tools/dist_check.py under torchrun."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_ham

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("key", ["m48_s12", "m64_s21", "m24_s100", "m32_s14", "m32_s6"])
def test_dist_path_single_gpu_matches_reference(key):
    from paper_2601_10557_b200 import SolverConfig
    from paper_2601_10557_b200.dist import solve_distributed

    kw = json.loads((GOLDEN / "meta.json").read_text())["cases"][key]
    m, seed = (int(t[1:]) for t in key.split("_"))
    a, b = golden_ham(m, seed)
    res = solve_distributed((a, b), SolverConfig(**kw), device=torch.device("cuda", 0))
    g = golden(f"solve_{key}.npz")
    assert res.converged == bool(g["converged"])
    assert abs(res.iterations_used - int(g["iterations_used"])) <= 1
    assert res.backup_events == int(g["backup_events"])
    if res.iterations_used == int(g["iterations_used"]):
        assert [t.variant for t in res.trace] == [str(x) for x in g["trace_variant"]]
    rel = np.abs(res.lambdas - g["lambdas"]) / np.abs(g["lambdas"])
    assert rel.max() <= 1e-10
    v = res.v.T.contiguous().cpu().numpy().T
    ov = np.abs(np.einsum("ij,ij->j", g["v"].conj(), v))
    assert np.abs(ov - 1).max() <= 1e-8


def test_start_block_device_policy_matches_host():
    """Above EXACT_LIMIT the start block comes from the device rng (generate.py's policy): same
    stream as the host draw (solver.py:139-141) to Box-Muller rounding, per-rank rows sliced right."""
    from paper_2601_10557_b200 import rng
    from paper_2601_10557_b200.dist import CudaOps, Grid, start_block_col
    from paper_2601_10557_b200.generate import EXACT_LIMIT

    m, cols, seed = EXACT_LIMIT + 3, 6, rng.substream(7, 3)
    n = 2 * m
    host = rng.complex_normal_matrix(seed, n, cols)
    dev = rng.device_complex_normal_matrix(seed, n, cols, torch.device("cuda", 0)).cpu().numpy()
    assert np.abs(dev - host).max() <= 1e-14 * np.abs(host).max()
    ops = CudaOps(torch.device("cuda", 0))
    for world, rank in ((2, 1), (4, 2), (8, 5)):
        g = Grid(m, world, rank)
        got = start_block_col(seed, n, cols, g, ops).cpu().numpy()  # (cols, 2 nc) storage
        rows = np.concatenate([np.arange(g.c0, g.c1), m + np.arange(g.c0, g.c1)])
        assert np.abs(got - host[rows].T).max() <= 1e-14 * np.abs(host).max()


def test_dist_c64_filter_matches_single_gpu_c64():
    """DistSolver.chebyshev_c64 on one GPU (tile kernel in raw mode, split, the grid's planes built
    from the transposed tile) is bitwise the single-GPU complex64 filter (bse_chebyshev_filter_c64),
    and within the FP32 accuracy of the FP64 filter."""
    from paper_2601_10557_b200 import rng
    from paper_2601_10557_b200.chebyshev import FilterConfig, filter_inplace
    from paper_2601_10557_b200 import BseHamiltonian, _lib
    from paper_2601_10557_b200.dist import DistributedSolver
    from paper_2601_10557_b200.hamiltonian import colmajor_empty

    dev = torch.device("cuda", 0)
    a, b = golden_ham(64, 21)
    m, n, k = 64, 128, 70
    ham = BseHamiltonian(a, b)
    fcfg = FilterConfig(10, 300.0, 250.0, -600.0)
    v0 = torch.from_numpy(rng.complex_normal_matrix(rng.substream(5, 3), n, k)).to(dev)
    single = colmajor_empty(n, k, dev)
    single.copy_(v0)
    prec = _lib.filter_precision()
    try:
        _lib.set_filter_precision("c64")
        filter_inplace(ham, single, fcfg)
    finally:
        _lib.set_filter_precision(prec)
    ds = DistributedSolver((a, b), device=dev, planes=False)  # c64 planes from the exact complex tiles
    vd = v0.T.contiguous()  # (k, n) storage = col layout at world 1
    ds.inner.chebyshev_c64(vd, fcfg)
    assert torch.equal(vd.T.cpu(), single.cpu())
    v128 = v0.T.contiguous()
    ds.inner.chebyshev(v128, fcfg, ds.inner.ops.empty(k, n))
    err = ((vd - v128).abs().amax(dim=1) / v128.abs().amax(dim=1)).max().item()
    assert err <= 2e-5, err


@pytest.mark.parametrize("pair", ["0", "1"])
def test_dist_c64_filter_b_zero(monkeypatch, pair):
    """B = 0 (the TDA limit, BSE_HAM_B_ZERO: the B half of the contraction is skipped) through the
    complex64 grid filter, single-CTA and CTA-pair kernels: within FP32 accuracy of the FP64 filter."""
    from paper_2601_10557_b200 import rng
    from paper_2601_10557_b200.chebyshev import FilterConfig
    from paper_2601_10557_b200.dist import DistributedSolver

    monkeypatch.setenv("BSE200_C64_PAIR", pair)
    dev = torch.device("cuda", 0)
    a, _ = golden_ham(64, 21)
    b = np.zeros_like(a)
    k = 70
    ds = DistributedSolver((a, b), device=dev)
    assert ds.flags & 1  # B == 0 detected
    ds.inner.ops.ctx.set_ham_flags(ds.flags)
    fcfg = FilterConfig(10, 300.0, 250.0, -600.0)
    v0 = torch.from_numpy(rng.complex_normal_matrix(rng.substream(9, 3), 128, k)).to(dev).T.contiguous()
    v64, v128 = v0.clone(), v0.clone()
    ds.inner.chebyshev_c64(v64, fcfg)
    ds.inner.chebyshev(v128, fcfg, ds.inner.ops.empty(k, 128))
    err = ((v64 - v128).abs().amax(dim=1) / v128.abs().amax(dim=1)).max().item()
    assert err <= 2e-5, err


@pytest.mark.parametrize("mr,kc,k", [(203, 157, 530), (157, 203, 100), (64, 64, 33), (9, 5, 1)])
def test_transposed_rs_product_from_forward_planes(mr, kc, k):
    """bse_hop_tile_rs_t on the planes of (A, B)[R, C] is BITWISE the forward real-split product on
    the planes of the explicit block transpose (A^H, B^T)[C, R] (Z' = -W^T, V' = V^T, U' = U^T,
    W' = -Z^T; hop_rs.cuh): the grid's row -> col step needs no second copy of the operator.
    Ragged shapes, both CTA tiles (k >= 512 / < 512), shift rows, beta term."""
    from paper_2601_10557_b200.dist import CudaOps, Tile, plane_tiles, tile_from_blocks

    dev = torch.device("cuda", 0)
    ops = CudaOps(dev)
    ops.ctx.set_ham_flags(0)
    gen = torch.Generator(device=dev).manual_seed(mr * 7 + kc)

    def rnd(*shape):
        return torch.complex(torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64),
                             torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64))

    a_t, b_t = rnd(mr, kc), rnd(mr, kc)  # any tile of a hermitian A / symmetric B
    fwd, trn = plane_tiles(ops, tile_from_blocks(ops, a_t, b_t))
    ref_f, _ = plane_tiles(ops, tile_from_blocks(ops, a_t, b_t, transpose=True))  # explicit transpose
    assert (trn.mr, trn.kc) == (kc, mr) and trn.trans and trn.g is fwd.g
    x = rnd(k, 2 * mr)  # folded input rows of the transposed product (contraction mr)
    p = rnd(k, 2 * kc)
    lo, hi = (2, min(mr, kc) - 1)
    out = {}
    for name, tile in (("trans", trn), ("explicit", ref_f)):
        y = torch.zeros(k, 2 * kc, dtype=torch.complex128, device=dev)
        ops.hop(tile, x, y, alpha=0.75, shift=3.5, shift_rows=(lo, hi), s_off=1, beta=0.25, p=p, filter=True,
                rs=True)
        out[name] = y
    torch.cuda.synchronize()
    assert torch.equal(out["trans"], out["explicit"])
    # and against the complex definition: x' = i Z' x + V' y, y' = U' x + i W' y with the transpose's planes
    at, bt = a_t.conj().T, b_t.T
    z, v, u, w = at.imag + bt.imag, at.real - bt.real, at.real + bt.real, at.imag - bt.imag
    xf, yf = x[:, :mr].T, x[:, mr:].T
    up = 1j * (z.to(xf.dtype) @ xf) + v.to(xf.dtype) @ yf
    low = u.to(xf.dtype) @ xf + 1j * (w.to(xf.dtype) @ yf)
    up[lo:hi] -= 3.5 * xf[lo + 1:hi + 1]
    low[lo:hi] -= 3.5 * yf[lo + 1:hi + 1]
    ref = torch.cat([0.75 * up - 0.25 * p[:, :kc].T, 0.75 * low - 0.25 * p[:, kc:].T]).T
    err = (out["trans"] - ref).abs().max().item() / ref.abs().max().item()
    assert err <= 1e-13, err


def test_grid_storage_is_one_tile_of_planes():
    """The real-split grid storage: one tile's planes per GPU (32 mr kc bytes), no complex tile."""
    from paper_2601_10557_b200.dist import DistributedSolver

    a, b = golden_ham(64, 21)
    ds = DistributedSolver((a, b), device=torch.device("cuda", 0))
    assert ds.planes and ds.fwd.buf is None and ds.trn.buf is None and ds.trn.g is ds.fwd.g
    assert ds.operator_bytes() == 4 * 64 * 64 * 8


@pytest.mark.parametrize("algo", ["rs", "rs-tall4-k32-split"])
@pytest.mark.parametrize("trans", [False, True])
def test_push_targets_and_group_sum(algo, trans):
    """The fused group reduction's device half on one GPU (dist.py _fused_reduce, BSE200_FUSED_REDUCE):
    with two push targets the real-split tile product (unsplit and split-K) stores its output into
    both inbox slots and not into y; bse_group_sum adds the slots in order.  Two copies of the same
    partial sum to exactly twice the pushed tile, which is the plain product's output to rounding."""
    import ctypes

    from paper_2601_10557_b200 import _lib
    from paper_2601_10557_b200.dist import CudaOps, plane_tiles, tile_from_blocks

    dev = torch.device("cuda", 0)
    ops = CudaOps(dev)
    ctx = ops.ctx
    ctx.set_ham_flags(0)
    gen = torch.Generator(device=dev).manual_seed(31)

    def rnd(*shape):
        return torch.complex(torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64),
                             torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64))

    mr, kc, k = 203, 157, 75
    fwd, trn = plane_tiles(ops, tile_from_blocks(ops, rnd(mr, kc), rnd(mr, kc)))
    tile = trn if trans else fwd
    rows_in, rows_out = (mr, kc) if trans else (kc, mr)
    x, p = rnd(k, 2 * rows_in), rnd(k, 2 * rows_out)
    kw = dict(alpha=0.75, shift=3.5, shift_rows=(1, min(mr, kc) - 1), s_off=1, beta=0.25, p=p, filter=True, rs=True)
    default = _lib.filter_algorithm()
    try:
        _lib.set_filter_algorithm(algo)
        ref = torch.zeros(k, 2 * rows_out, dtype=torch.complex128, device=dev)
        ops.hop(tile, x, ref, **kw)
        cap = k * 2 * rows_out + 64  # slot stride larger than the block, as for a full-width inbox
        inbox = torch.zeros(2 * cap, dtype=torch.complex128, device=dev)
        untouched = torch.full((k, 2 * rows_out), 7.0, dtype=torch.complex128, device=dev)
        targets = (ctypes.c_void_p * 2)(inbox.data_ptr(), inbox.data_ptr() + cap * 16)
        ctx.call("bse_set_push_targets", targets, 2)
        try:
            ops.hop(tile, x, untouched, **kw)
        finally:
            ctx.call("bse_set_push_targets", None, 0)
        out = torch.empty_like(ref)
        ctx.call("bse_group_sum", inbox.data_ptr(), cap, 2, out.data_ptr(), out.numel())
        torch.cuda.synchronize()
    finally:
        _lib.set_filter_algorithm(default)
    assert torch.equal(untouched, torch.full_like(untouched, 7.0))  # no local store while pushing
    s0 = inbox[:k * 2 * rows_out].view(k, -1)
    s1 = inbox[cap:cap + k * 2 * rows_out].view(k, -1)
    assert torch.equal(s0, s1)  # every target receives the same bits
    # the pushed tile equals the local-store product to rounding (the compiler may contract the
    # epilogue's multiply-adds differently on the two store paths)
    assert (s0 - ref).abs().max().item() <= 4e-16 * ref.abs().max().item()
    assert torch.equal(out, s0 + s1)
