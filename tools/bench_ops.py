"""Wall-clock breakdown of the non-filter operators at C2/C3 shapes (host overhead hunt),
and 4M vs 3M filter-step throughput."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2601_10557_b200 as bse
from paper_2601_10557_b200 import _lib
from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of
from paper_2601_10557_b200.ortho import s_orthonormalize_inplace
from paper_2601_10557_b200.rayleigh_ritz import build_hermitian_rq_device, residuals_device


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def main(m, k, l):
    dev = torch.device("cuda", 0)
    ham = bse.generate(bse.GeneratorSpec(m=m, seed=0))
    n = 2 * m
    v0 = colmajor_empty(n, k, dev)
    v0.real.normal_()
    v0.imag.normal_()
    y = colmajor_empty(n, l, dev)
    y.real.normal_()
    y.imag.normal_()
    y /= torch.linalg.vector_norm(y, dim=0)
    v = v0.clone()
    print(f"m={m} k={k} l={l}")
    print(f"  s_orthonormalize (l={l}): {wall(lambda: (v.copy_(v0), s_orthonormalize_inplace(v, y))):.1f} ms")
    print(f"  s_orthonormalize (l=0):   {wall(lambda: (v.copy_(v0), s_orthonormalize_inplace(v, None))):.1f} ms")
    v.copy_(v0)
    s_orthonormalize_inplace(v, None)
    print(f"  rr_hermitian:             {wall(lambda: build_hermitian_rq_device(ham, v)):.1f} ms")
    r, _ = build_hermitian_rq_device(ham, v)
    print(f"  residuals:                {wall(lambda: residuals_device(ham, r.values, r.vectors)):.1f} ms")
    ctx = _lib.Context.get(0)
    ab = ham.device_blocks(dev)
    t = colmajor_empty(n, k, dev)
    print(f"  apply_sh:                 {wall(lambda: ctx.call('bse_apply_h', _lib.dptr(ab), None, ld_of(ab), m, _lib.dptr(v), n, _lib.dptr(t), n, k, -1.0)):.1f} ms")
    w = torch.empty((k, k), dtype=torch.complex128, device=dev)
    g2 = torch.empty((k, k), dtype=torch.complex128, device=dev)
    wv = torch.empty((k, k), dtype=torch.complex128, device=dev)
    lam = np.zeros(k)
    import ctypes
    lmm = ctypes.c_double()

    def pencil():
        ctx.call("bse_zgemm_cn", k, k, n, 1.0, _lib.dptr(v), n, _lib.dptr(t), n, 0.0, _lib.dptr(w), k)
        ctx.call("bse_zgemm_cn", k, k, m, 1.0, v.data_ptr() + m * 16, n, v.data_ptr() + m * 16, n, 0.0, _lib.dptr(g2), k)
        ctx.call("bse_rr_pencil", _lib.dptr(w), _lib.dptr(g2), k, _lib.hptr(lam), _lib.dptr(wv), ctypes.byref(lmm))
    print(f"  grams + rr_pencil:        {wall(pencil):.1f} ms")
    wk = w.clone()
    print(f"  eigvalsh k x k:           {wall(lambda: ctx.call('bse_eigvalsh', _lib.dptr(wk), k, k, _lib.hptr(lam))):.1f} ms")
    for alg in ("4m", "3m", "rs"):
        bse.set_filter_algorithm(alg)
        sdp = _lib.dptr(ham.device_sum_planes(dev)) if alg == "3m" else None
        yp = v0.clone()
        yn = colmajor_empty(n, k, dev)
        ms = wall(lambda: ctx.call("bse_filter_step", _lib.dptr(ab), sdp, ld_of(ab), m, _lib.dptr(v), _lib.dptr(yp),
                                   _lib.dptr(yn), n, k, 0.1, 1e-3, 0.5), reps=3)
        print(f"  filter step {alg}: {ms:.1f} ms = {8.0 * n * n * k / ms / 1e9:.2f} TFLOP/s (model)")
    bse.set_filter_algorithm("4m")


if __name__ == "__main__":
    main(10000, 600, 300)
    main(20000, 1200, 600)
