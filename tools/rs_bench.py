"""Real-split filter kernel timing at the C3 operator size (m = 20,000): the forward product
(bse_chebyshev_filter_rs, per step) and the grid's transposed product (bse_hop_tile_rs_t) on the
same planes; executed TF/s (4 n^2 k per step) against the measured 37.1 TF/s DMMA peak.

    python tools/rs_bench.py [m] [k,k,...] [code,code,...]   (bse_set_filter_algorithm codes)

BSE200_RS_KSPLIT=s fixes the split-K factor of code 90 (0: planned per product; code 98 = tile 97, split 2).
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2601_10557_b200 import _lib
from paper_2601_10557_b200.dist import CudaOps, Tile, plane_tiles
from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of

PEAK = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())["dmma_tflops"]
m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1200, 300, 100]
codes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [90]
dev = torch.device("cuda", 0)
ops = CudaOps(dev)
ctx = ops.ctx
ctx.set_ham_flags(0)
n = 2 * m
ab = colmajor_empty(m, 2 * m, dev)
ab.real.normal_()
ab.imag.normal_()
addr = ab.data_ptr()
tile = Tile(ab, addr, addr + m * m * 16, m, m, m)
fwd, trn = plane_tiles(ops, tile)
del ab, tile
torch.cuda.empty_cache()


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = []
for k in ks:
    v0 = colmajor_empty(n, k, dev)
    v0.real.normal_()
    v0.imag.normal_()
    work = torch.empty(2 * n * k, dtype=torch.complex128, device=dev)
    x = torch.empty((k, n), dtype=torch.complex128, device=dev)
    x.real.normal_()
    x.imag.normal_()
    y = torch.empty_like(x)
    deg = 4
    ref = None
    for code in codes:
        ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, code))
        v = v0.clone()
        ms_f = timed(lambda: ctx.call("bse_chebyshev_filter_rs", fwd.g.data_ptr(), fwd.ldg, m, _lib.dptr(v), n, k, deg,
                                      0.0, 1.0, -1.5, _lib.dptr(work)), 2) / deg
        ms_t = timed(lambda: ops.hop(trn, x, y, alpha=0.5, shift=0.1, shift_rows=(0, m), s_off=0, filter=True,
                                     rs=True), 4)
        yy = y.clone()
        same = None if ref is None else bool(torch.equal(ref, yy))
        rdiff = None if ref is None else float((yy - ref).abs().max() / ref.abs().max())
        ref = yy if ref is None else ref
        ex = 4.0 * n * n * k / 1e12
        row = {"m": m, "k": k, "code": code, "fwd_ms": ms_f, "fwd_tflops": ex / ms_f * 1e3,
               "fwd_frac": ex / ms_f * 1e3 / PEAK, "trans_ms": ms_t, "trans_tflops": ex / ms_t * 1e3,
               "trans_frac": ex / ms_t * 1e3 / PEAK, "bitwise_as_first_code": same,
               "max_rel_diff_vs_first": rdiff}
        out.append(row)
        print(json.dumps({kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in row.items()}), flush=True)
ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, 90))
