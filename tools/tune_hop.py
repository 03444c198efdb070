"""Filter-step kernel variants (bse_set_filter_algorithm codes) and small-k cuSOLVER timings."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_10557_b200 import _lib
from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of

ctx = _lib.Context.get(0)
dev = torch.device("cuda", 0)


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


def variants(m, ks, codes):
    n = 2 * m
    ab = colmajor_empty(m, 2 * m, dev)
    ab.real.normal_()
    ab.imag.normal_()
    sd = colmajor_empty(m, 2 * m, dev)
    ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m, _lib.dptr(sd))
    for k in ks:
        y = colmajor_empty(n, k, dev); y.real.normal_(); y.imag.normal_()
        yp = colmajor_empty(n, k, dev); yp.real.normal_(); yp.imag.normal_()
        yn = colmajor_empty(n, k, dev)
        for code in codes:
            ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, code))
            sdp = _lib.dptr(sd) if code in (6, 7, 8, 81) or 61 <= code <= 63 else None
            ms = timed(lambda: ctx.call("bse_filter_step", _lib.dptr(ab), sdp, ld_of(ab), m, _lib.dptr(y), _lib.dptr(yp),
                                        _lib.dptr(yn), n, k, 0.1, 1e-3, 0.5), 3 if m >= 20000 else 5)
            tf = 8.0 * n * n * k / ms / 1e9
            cm = 3 if code in (3, 31, 32, 33, 34, 6, 61, 62, 63) else 4
            print(f"m={m} k={k} code={code}: {ms:8.2f} ms  model {tf:6.2f} TF/s  executed {tf * (0.75 if cm == 3 else 1):6.2f}",
                  flush=True)
    ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, 4))


def whole_filter(m, ks, codes, deg=4):
    """bse_chebyshev_filter (deg steps) per filter code — codes 6/7 get the sum planes."""
    n = 2 * m
    ab = colmajor_empty(m, 2 * m, dev)
    ab.real.normal_()
    ab.imag.normal_()
    sd = colmajor_empty(m, 2 * m, dev)
    ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m, _lib.dptr(sd))
    for k in ks:
        v = colmajor_empty(n, k, dev); v.real.normal_(); v.imag.normal_()
        work = torch.empty(2 * n * k, dtype=torch.complex128, device=dev)
        for code in codes:
            ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, code))
            sdp = _lib.dptr(sd) if code in (82, 86, 88) else None
            ms = timed(lambda: ctx.call("bse_chebyshev_filter", _lib.dptr(ab), sdp, ld_of(ab), m, _lib.dptr(v), n, k,
                                        deg, 0.0, 1.0, -1.5, _lib.dptr(work)), 2)
            print(f"filter deg={deg} m={m} k={k} code={code}: {ms / deg:8.2f} ms/step  model "
                  f"{8.0 * n * n * k * deg / ms / 1e9:6.2f} TF/s", flush=True)
    ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, 88))


def c64_filter(m, ks, deg=4):
    """bse_chebyshev_filter_c64 (tcgen05 3xTF32) per step."""
    n = 2 * m
    mp = (m + 3) // 4 * 4
    ab = colmajor_empty(m, 2 * m, dev)
    ab.real.normal_()
    ab.imag.normal_()
    pl = torch.empty(4 * m * 2 * mp, dtype=torch.float32, device=dev)
    ctx.call("bse_c64_prepare", _lib.dptr(ab), ld_of(ab), m, _lib.dptr(pl))
    for k in ks:
        v = colmajor_empty(n, k, dev); v.real.normal_(); v.imag.normal_()
        work = torch.empty(48 * mp * k, dtype=torch.float32, device=dev)
        ms = timed(lambda: ctx.call("bse_chebyshev_filter_c64", _lib.dptr(pl), m, _lib.dptr(v), n, k, deg, 0.0, 1.0,
                                    -1.5, _lib.dptr(work)), 2)
        print(f"c64 filter deg={deg} m={m} k={k}: {ms / deg:8.2f} ms/step  model {8.0 * n * n * k * deg / ms / 1e9:7.1f} "
              f"TF/s  (tf32 executed {3 * 8.0 * n * n * k * deg / ms / 1e9:7.1f})", flush=True)


def solver_small():
    for k in (100, 200, 400, 600, 800, 1000, 1200):
        g = torch.randn((k, k), dtype=torch.complex128, device=dev)
        g = g @ g.conj().T / k + torch.eye(k, dtype=torch.complex128, device=dev)
        w = np.zeros(k)
        lam = np.zeros(k)
        wv = torch.empty_like(g)
        lmm = ctypes.c_double()
        t0 = time.perf_counter()
        ctx.call("bse_eigvalsh", _lib.dptr(g), k, k, _lib.hptr(w))
        t1 = time.perf_counter()
        g2 = 0.25 * torch.eye(k, dtype=torch.complex128, device=dev) + 0.01 * (g - torch.eye(k, dtype=g.dtype, device=dev))
        wm = g.clone()
        t2 = time.perf_counter()
        ctx.call("bse_rr_pencil", _lib.dptr(wm), _lib.dptr(g2.clone()), k, _lib.hptr(lam), _lib.dptr(wv), ctypes.byref(lmm))
        t3 = time.perf_counter()
        wm = g.clone()
        t4 = time.perf_counter()
        ctx.call("bse_rr_pencil", _lib.dptr(wm), _lib.dptr(g2.clone()), k, _lib.hptr(lam), _lib.dptr(wv), ctypes.byref(lmm))
        t5 = time.perf_counter()
        print(f"k={k}: eigvalsh {1e3 * (t1 - t0):.1f} ms, rr_pencil {1e3 * (t3 - t2):.1f} ms / again {1e3 * (t5 - t4):.1f} ms",
              flush=True)


if __name__ == "__main__":
    solver_small()
    variants(20000, [1200, 300], [4, 41, 42, 43, 3, 31, 32, 33, 34])
    variants(10000, [600, 113], [4, 41, 42, 43, 3, 31, 32, 33, 34])
