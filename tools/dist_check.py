"""Multi-GPU parity check of the 2D-distributed solve (run under torchrun, NCCL):
golden reference cases + C1, compared on rank 0 with the reference fixtures.

BSE200_DIST_BACKEND=gloo runs more ranks than GPUs (rank r on GPU r % #GPUs, gloo collectives on
the CUDA tensors): the 2 x 4 grid of an 8-GPU box with the real CUDA kernels on a 4-GPU box."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch
import torch.distributed as dist

from conftest import GOLDEN, golden, golden_ham, rebuild_c1
from paper_2601_10557_b200 import SolverConfig
from paper_2601_10557_b200.dist import DistSolver, solve_distributed

DistSolver.CHUNK_MIN = 8  # exercise the chunked, stream-overlapped filter on the small cases


def main():
    backend = os.environ.get("BSE200_DIST_BACKEND", "nccl")
    local = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
        DistSolver.CHUNK_MIN = 1 << 30  # no communication-stream overlap under gloo
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    fails = 0
    cases = json.loads((GOLDEN / "meta.json").read_text())["cases"]
    for key in ["m48_s12", "m64_s21", "m24_s100", "m32_s14", "m48_s13", "m32_s6"]:
        m, seed = (int(t[1:]) for t in key.split("_"))
        a, b = golden_ham(m, seed)
        res = solve_distributed((a, b), SolverConfig(**cases[key]), device=dev)
        if rank == 0:
            g = golden(f"solve_{key}.npz")
            rel = float(np.max(np.abs(res.lambdas - g["lambdas"]) / np.abs(g["lambdas"])))
            v = res.v.T.contiguous().cpu().numpy().T
            ov = float(np.abs(np.abs(np.einsum("ij,ij->j", g["v"].conj(), v)) - 1).max())
            ok = rel <= 1e-10 and ov <= 1e-8 and abs(res.iterations_used - int(g["iterations_used"])) <= 1
            fails += not ok
            print(f"[world {world}] {key}: iters {res.iterations_used}/{int(g['iterations_used'])} "
                  f"max rel dlambda {rel:.2e} subspace {ov:.2e} {'OK' if ok else 'FAIL'}", flush=True)
    # complex64 filter on the grid (raw partials -> fp32 allreduce -> split) vs the FP64 filter
    from paper_2601_10557_b200 import rng as _rng
    from paper_2601_10557_b200.chebyshev import FilterConfig
    from paper_2601_10557_b200.dist import DistributedSolver, start_block_col

    a, b = golden_ham(64, 21)
    ds = DistributedSolver((a, b), device=dev)
    fcfg = FilterConfig(10, 300.0, 250.0, -600.0)
    v = start_block_col(_rng.substream(5, 3), 128, 70, ds.inner.g, ds.inner.ops)
    v64 = v.clone()
    ds.inner.chebyshev(v, fcfg, ds.inner.ops.empty(70, 2 * ds.inner.g.nr))
    ds.inner.chebyshev_c64(v64, fcfg)
    f128, f64 = ds.inner.assemble_from_col(v), ds.inner.assemble_from_col(v64)
    if rank == 0:
        err = float(((f64 - f128).abs().amax(dim=1) / f128.abs().amax(dim=1)).max())
        ok = err <= 2e-5
        fails += not ok
        print(f"[world {world}] c64 filter vs FP64 (m=64, deg 10): max rel {err:.2e} {'OK' if ok else 'FAIL'}",
              flush=True)
    # mixed-precision policy (complex64 filters while residuals are large) on the grid
    from paper_2601_10557_b200.solver import set_mixed_precision

    set_mixed_precision(True)
    try:
        a, b, g = rebuild_c1()
        res = solve_distributed((a, b), SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0), device=dev)
    finally:
        set_mixed_precision(False)
    if rank == 0:
        rel = float(np.max(np.abs(res.lambdas - g["abs_lambdas"]) / np.abs(g["abs_lambdas"])))
        ok = rel <= 1e-10 and res.converged and res.residual_norms.max() <= 1e-10 and "c64" in res.filter_precisions
        fails += not ok
        print(f"[world {world}] C1 mixed policy: iters {res.iterations_used} filters {''.join(p[1] for p in res.filter_precisions)} "
              f"max rel dlambda {rel:.2e} {'OK' if ok else 'FAIL'}", flush=True)
    a, b, g = rebuild_c1()
    res = solve_distributed((a, b), SolverConfig(nev=50, nex=20, deg=20, tol=1e-10, seed=0), device=dev)
    if rank == 0:
        rel = float(np.max(np.abs(res.lambdas - g["abs_lambdas"]) / np.abs(g["abs_lambdas"])))
        ok = rel <= 1e-10 and res.converged and abs(res.iterations_used - int(g["abs_iters"])) <= 1 \
            and res.residual_norms.max() <= 1e-10
        fails += not ok
        print(f"[world {world}] C1 m=500: iters {res.iterations_used}/{int(g['abs_iters'])} max rel dlambda "
              f"{rel:.2e} max res {res.residual_norms.max():.2e} {'OK' if ok else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
