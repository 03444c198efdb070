"""Kernel-level breakdown of one solve with torch.profiler (CUPTI): which kernels
(ours, cuSOLVER, cuBLAS, torch copies) take the device time outside the filter."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2601_10557_b200 as bse

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
m, nev, nex = {"c2": (10000, 500, 100), "c3": (20000, 1000, 200), "c1": (500, 50, 20)}[cfgname]
ham = bse.generate(bse.GeneratorSpec(m=m, seed=0))
cfg = bse.SolverConfig(nev=nev, nex=nex, deg=20, tol=1e-10, seed=0, rel_res=cfgname != "c1")
bse.solve(ham, cfg, keep_on_device=True)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = bse.solve(ham, cfg, keep_on_device=True)
print("ledger seconds", {k: round(v, 3) for k, v in r.ledger.seconds.items()}, "iters", r.iterations_used)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=90))
