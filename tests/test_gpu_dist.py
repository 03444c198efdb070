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
    ds = DistributedSolver((a, b), device=dev)
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
