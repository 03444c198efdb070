"""Real-split filter (csrc/hop_rs.cuh, codes 90-94) vs the default 3M TMA filter (88) at the C3
operator size: ms per Chebyshev step, model (8 n^2 k) and executed TF/s, and the max difference
of the filtered block against 3M relative to its scale."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import tune_hop
from tune_hop import ctx, dev, timed, colmajor_empty, ld_of, _lib

m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1200, 600, 300, 100]
codes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [88, 90, 91, 92, 93, 94]
deg = 4
n = 2 * m
ab = colmajor_empty(m, 2 * m, dev); ab.real.normal_(); ab.imag.normal_()
sd = colmajor_empty(m, 2 * m, dev)
ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m, _lib.dptr(sd))
ldg = m + (m & 1)
gp = torch.empty((4 * m, ldg), dtype=torch.float64, device=dev).t()
ctx.call("bse_make_rs_planes", _lib.dptr(ab), ld_of(ab), m, m, _lib.dptr(gp), ldg)
for k in ks:
    v0 = colmajor_empty(n, k, dev); v0.real.normal_(); v0.imag.normal_()
    work = torch.empty(2 * n * k, dtype=torch.complex128, device=dev)
    ref = None
    for code in codes:
        ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, code))
        v = v0.clone()
        if code >= 90:
            fn = lambda: ctx.call("bse_chebyshev_filter_rs", _lib.dptr(gp), ldg, m, _lib.dptr(v), n, k, deg, 0.0, 1.0,
                                  -1.5, _lib.dptr(work))
        else:
            fn = lambda: ctx.call("bse_chebyshev_filter", _lib.dptr(ab), _lib.dptr(sd), ld_of(ab), m, _lib.dptr(v), n, k,
                                  deg, 0.0, 1.0, -1.5, _lib.dptr(work))
        v.copy_(v0)
        fn()
        torch.cuda.synchronize()
        out = v.clone()
        if ref is None:
            ref = out
        diff = ((out - ref).abs().max() / ref.abs().max()).item()
        ms = timed(fn, 2) / deg
        mod = 8.0 * n * n * k / ms / 1e9
        ex = mod * (0.5 if code >= 90 else 0.75)
        print(f"m={m} k={k} code={code}: {ms:8.2f} ms/step  model {mod:6.2f} TF/s  executed {ex:6.2f} TF/s  "
              f"rel diff vs first {diff:.2e}", flush=True)
ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, 88))
