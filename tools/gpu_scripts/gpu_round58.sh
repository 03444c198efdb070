#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hbm_is_short or bitwise" 2>&1 | tail -2
cat > /tmp/np.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import torch
import tune_hop
from tune_hop import ctx, dev, timed, colmajor_empty, ld_of, _lib
m, deg = 20000, 4
n = 2 * m
ab = colmajor_empty(m, 2 * m, dev); ab.real.normal_(); ab.imag.normal_()
sd = colmajor_empty(m, 2 * m, dev)
ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m, _lib.dptr(sd))
ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, 88))
for k in (1200, 300):
    v = colmajor_empty(n, k, dev); v.real.normal_(); v.imag.normal_()
    work = torch.empty(2 * n * k, dtype=torch.complex128, device=dev)
    for label, sdp in (("planes (88)", _lib.dptr(sd)), ("registers (98)", None)):
        ms = timed(lambda: ctx.call("bse_chebyshev_filter", _lib.dptr(ab), sdp, ld_of(ab), m, _lib.dptr(v), n, k, deg,
                                    0.0, 1.0, -1.5, _lib.dptr(work)), 2)
        print(f"filter k={k} {label}: {ms / deg:8.2f} ms/step  model {8.0 * n * n * k * deg / ms / 1e9:6.2f} TF/s", flush=True)
PY
timeout 600 python /tmp/np.py 2>&1 | tail -4
