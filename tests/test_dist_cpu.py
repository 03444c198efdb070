"""2D-distributed solve (paper_2601_10557_b200/dist.py) on CPU under gloo with
world_size 1, 2 and 4 (torch reference ops in place of the CUDA kernels),
against the reference golden fixtures."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import GOLDEN, golden, golden_ham


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, key, pq, out, planes=None):
    import torch.distributed as dist
    from dist_torch_ops import TorchOps
    from paper_2601_10557_b200 import SolverConfig
    from paper_2601_10557_b200.dist import Grid, solve_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    kw = json.loads((GOLDEN / "meta.json").read_text())["cases"][key]
    m, seed = (int(t[1:]) for t in key.split("_"))
    a, b = golden_ham(m, seed)
    grid = Grid(m, world, rank, *pq) if pq else None
    from paper_2601_10557_b200.dist import DistSolver

    DistSolver.CHUNK_MIN = 4  # exercise the column-chunked filter pipeline on the small cases
    DistSolver.START_SPLIT_MIN = 4  # and the two-half start block / first filter
    from paper_2601_10557_b200.dist import DistributedSolver as DS

    ds = DS((a, b), device=torch.device("cpu"), grid=grid, ops=TorchOps(), planes=planes)
    assert ds.planes == (planes is not False and not ds.flags & 1)  # B = 0 keeps the complex tiles
    res = ds.solve(SolverConfig(**kw))
    if rank == 0:
        np.savez(out, lambdas=res.lambdas, v=res.v.numpy(), res=res.residual_norms, iters=res.iterations_used,
                 converged=res.converged, locked=[t.locked for t in res.trace], k=[t.k for t in res.trace],
                 variant=[t.variant for t in res.trace], flops=[t.flops for t in res.trace],
                 backups=res.backup_events)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,pq,key,planes", [
    (1, None, "m48_s12", None), (2, None, "m48_s12", None), (4, None, "m64_s21", None),
    (2, (2, 1), "m24_s100", None), (4, (1, 4), "m32_s14", None), (8, None, "m64_s40", None),
    (2, None, "m32_s6", None), (4, None, "m32_s6", None), (8, None, "m48_s13", None),
    # complex tiles + block transposes (B = 0 storage) on B != 0 inputs
    (4, None, "m64_s21", False), (8, None, "m48_s12", False)])
def test_distributed_solve_matches_reference(tmp_path, world, pq, key, planes):
    """planes=None: the default real-split storage (one tile's planes per rank, the transposed
    product read from them); False: complex tiles.  Same bar as the single-GPU golden solves."""
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _port(), key, pq, out, planes), nprocs=world, join=True)
    r = np.load(out)
    g = golden(f"solve_{key}.npz")
    assert bool(r["converged"]) == bool(g["converged"])
    assert abs(int(r["iters"]) - int(g["iterations_used"])) <= 1
    if int(r["iters"]) == int(g["iterations_used"]):
        assert list(r["locked"]) == list(g["trace_locked"])
        assert list(r["variant"]) == [str(x) for x in g["trace_variant"]]
        np.testing.assert_allclose(r["flops"], g["trace_flops"], rtol=1e-12)
    assert int(r["backups"]) == int(g["backup_events"])
    rel = np.abs(r["lambdas"] - g["lambdas"]) / np.abs(g["lambdas"])
    assert rel.max() <= 1e-10
    ov = np.abs(np.einsum("ij,ij->j", g["v"].conj(), r["v"]))
    assert np.abs(ov - 1).max() <= 1e-8


def test_grid_shapes_and_diag_cover():
    from paper_2601_10557_b200.dist import Grid, grid_shape

    assert [grid_shape(w) for w in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
    for world in (1, 2, 4, 8):
        for m in (7, 40, 101):
            grids = [Grid(m, world, r) for r in range(world)]
            p, q = grids[0].p, grids[0].q
            for I in range(p):  # each output row of a row group is shifted exactly once
                cover = np.zeros(m, int)
                for gr in grids[I * q:(I + 1) * q]:
                    lo, hi = gr.diag
                    cover[lo:hi] += 1
                assert (cover[gr.r0:gr.r1] == 1).all() and cover.sum() == gr.nr


def _c64_worker(rank, world, port, out):
    import torch.distributed as dist
    from dist_torch_ops import TorchOps
    from paper_2601_10557_b200 import rng
    from paper_2601_10557_b200.chebyshev import FilterConfig
    from paper_2601_10557_b200.dist import DistributedSolver, start_block_col
    from paper_2601_10557_b200.metrics import PhaseLedger

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    a, b = golden_ham(48, 12)
    ops = TorchOps()
    ds = DistributedSolver((a, b), device=torch.device("cpu"), ops=ops)
    inner = ds.inner
    g = inner.g
    bounds = inner.lanczos(12, 24, rng.substream(12, 2), PhaseLedger())
    fcfg = FilterConfig.from_bounds(bounds, 10, False)
    v = start_block_col(rng.substream(12, 3), 96, 12, g, ops)
    v64 = v.clone()
    inner.chebyshev(v, fcfg, ops.empty(12, 2 * g.nr))
    inner.chebyshev_c64(v64, fcfg)
    f128, f64 = inner.assemble_from_col(v), inner.assemble_from_col(v64)
    if rank == 0:
        np.savez(out, f128=f128.numpy(), f64=f64.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_distributed_c64_filter_matches_fp64(tmp_path, world):
    """dist.DistSolver.chebyshev_c64 (raw partials -> allreduce -> split, beta on the reduction
    group's owner, shift on the diagonal rows) against the FP64 distributed filter: equal to the
    complex64 rounding of each step (deg 10, columns scaled by their norm)."""
    out = str(tmp_path / "c.npz")
    mp.spawn(_c64_worker, args=(world, _port(), out), nprocs=world, join=True)
    r = np.load(out)
    f128, f64 = r["f128"], r["f64"]
    err = np.abs(f64 - f128).max(axis=1) / np.abs(f128).max(axis=1)
    assert err.max() <= 2e-5, err.max()


def _phase_worker(rank, world, port, out):
    import torch.distributed as dist
    from dist_torch_ops import TorchOps
    from paper_2601_10557_b200 import rng
    from paper_2601_10557_b200.dist import DistributedSolver, start_block_col

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    a, b = golden_ham(48, 12)
    ops = TorchOps()
    ds = DistributedSolver((a, b), device=torch.device("cpu"), ops=ops)
    g = ds.inner.g
    q = start_block_col(rng.substream(4, 3), 96, 9, g, ops)
    q[:, :2] = 0.0  # leading zero rows of this rank's upper-half slice: the "first" entry moves
    q[5] = 0.0  # a zero column stays untouched
    ds.inner.fix_phases(q)
    full = ds.inner.assemble_from_col(q)
    if rank == 0:
        np.save(out, full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_distributed_phase_convention(tmp_path, world):
    """dist.DistSolver.fix_phases == ortho.py:70-82 on the assembled block (first entry with
    |q| >= 1e-8 max|q| in global row order made real positive; zero columns untouched)."""
    from oracle import bse_oracle as o
    from paper_2601_10557_b200 import rng

    out = str(tmp_path / "q.npy")
    mp.spawn(_phase_worker, args=(world, _port(), out), nprocs=world, join=True)
    got = np.load(out).T
    raw = rng.complex_normal_matrix(rng.substream(4, 3), 96, 9)
    from paper_2601_10557_b200.dist import Grid

    ref_in = raw.copy()  # the same input, assembled: each rank zeroed 2 rows of its upper slice
    for r in range(world):
        gr = Grid(48, world, r)
        ref_in[gr.c0:min(gr.c0 + 2, gr.c1)] = 0.0
    ref_in[:, 5] = 0.0
    ref = o.phase_fix(ref_in)
    assert np.abs(got - ref).max() <= 1e-15
