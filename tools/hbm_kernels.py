"""Achieved HBM bandwidth of the memory-bound kernels on the solve path (north star: "achieved HBM
GB/s for the QR, residual and axpby kernels"), at C3 shapes (m = 20000, n = 40000, k = 1200),
timed with CUDA events on the library's stream (torch's current stream), L2 flushed before
every timed call, against MEASURED_PEAKS.json's HBM figure.

The axpby of the Chebyshev recurrence and the S-flip of the RR product are fused into the GEMM
epilogues (no standalone pass); the standalone HBM-bound kernels are the ones below.
Bytes are algorithmic (each operand read / written once).  Run: python tools/hbm_kernels.py"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_10557_b200 import _lib
from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of

PEAK = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6553.9


_FLUSH = None


def timed(fn, reps=10):
    """Median of reps CUDA-event timings, the 126 MB L2 flushed (a 512 MB write) before each."""
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        _FLUSH.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main(m=20000, k=1200):
    dev = torch.device("cuda", 0)
    ctx = _lib.Context.get(0)
    n = 2 * m
    rows = []

    def report(name, ms, nbytes, what):
        gbs = nbytes / (ms * 1e-3) / 1e9
        rows.append({"kernel": name, "ms": round(ms, 4), "bytes": int(nbytes), "GB/s": round(gbs, 1),
                     "frac_of_hbm_peak": round(gbs / PEAK, 3), "what": what})
        print(f"{name:34s} {ms:8.3f} ms  {nbytes / 1e9:8.3f} GB  {gbs:8.1f} GB/s  {gbs / PEAK:6.1%}  {what}",
              flush=True)

    x = colmajor_empty(n, k, dev)
    x.real.normal_()
    x.imag.normal_()
    y = colmajor_empty(n, k, dev)
    y.copy_(x)
    out = torch.empty(k, dtype=torch.float64, device=dev)
    lam = torch.randn(k, dtype=torch.float64, device=dev)
    ones = torch.ones(k, dtype=torch.float64, device=dev)
    nrm = torch.full((k,), 4.0, dtype=torch.float64, device=dev)

    report("colnorm2 (frob2_kernel)", timed(lambda: ctx.call("bse_colnorm2", _lib.dptr(x), n, k, ld_of(x), _lib.dptr(out))),
           16 * n * k, "squared column norms of V (normalise Ritz vectors, CholQR3 shift): read n k")
    report("colscale_rsqrt (colscale_inv)", timed(lambda: ctx.call("bse_colscale_rsqrt", _lib.dptr(y), n, k, ld_of(y),
                                                                    _lib.dptr(nrm))),
           32 * n * k, "V /= |V| per column: read + write n k")
    report("resid_partial (resid_from_rr)", timed(lambda: ctx.call("bse_resid_partial", _lib.dptr(x), ld_of(x), _lib.dptr(y),
                                                                    ld_of(y), n, m, k, _lib.dptr(ones), _lib.dptr(lam),
                                                                    _lib.dptr(out))),
           32 * n * k, "||S (S H Q) w / |Q w| - lam v||^2 partials: read 2 n k")
    report("sflip", timed(lambda: ctx.call("bse_sflip", _lib.dptr(x), ld_of(x), _lib.dptr(y), ld_of(y), m, k)),
           32 * n * k, "y = S x (basis of span(S Y_locked)): read + write n k")
    report("fix_phases (phase_fix)", timed(lambda: ctx.call("bse_fix_phases", _lib.dptr(y), n, k, ld_of(y))),
           32 * n * k, "ortho.py:70-82 column phases: read + write n k (+ pivot scan)")
    ab = colmajor_empty(m, 2 * m, dev)
    ab.real.normal_()
    ab.imag.normal_()
    sd = colmajor_empty(m, 2 * m, dev)
    report("make_sum_planes", timed(lambda: ctx.call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), m, 2 * m,
                                                      _lib.dptr(sd)), reps=3),
           64 * m * m, "(Pr+Pi, Pr-Pi) planes of [A|B], once per Hamiltonian: read + write 32 m^2")
    xv = colmajor_empty(n, 1, dev)
    xv.real.normal_()
    xv.imag.normal_()
    yv = colmajor_empty(n, 1, dev)
    report("apply_h k=1 (gemv_partial+reduce)", timed(lambda: ctx.call("bse_apply_h", _lib.dptr(ab), None, ld_of(ab), m,
                                                                        _lib.dptr(xv), n, _lib.dptr(yv), n, 1, 1.0)),
           32 * m * m, "Lanczos matvec (lanczos.py:53-88): read [A|B] once")
    # CholQR Gram / update (ortho.py:115-119): compute-bound at k = 1200 (AI ~ k/2), reported as TF/s
    g = torch.empty((k, k), dtype=torch.complex128, device=dev)
    ms = timed(lambda: ctx.call("bse_zgemm_cn", k, k, n, 1.0, _lib.dptr(x), ld_of(x), _lib.dptr(x), ld_of(x), 0.0,
                                _lib.dptr(g), k), reps=5)
    print(f"{'gram Q^H Q (zgemm_cn, DMMA)':34s} {ms:8.3f} ms  {8.0 * n * k * k / ms / 1e9:8.2f} TFLOP/s (8 n k^2)")
    rows.append({"kernel": "gram Q^H Q (zgemm_cn)", "ms": round(ms, 4), "TFLOP/s": round(8.0 * n * k * k / ms / 1e9, 2),
                 "what": "CholQR Gram, compute-bound"})
    ms = timed(lambda: ctx.call("bse_zgemm_nn", n, k, k, 1.0, _lib.dptr(x), ld_of(x), _lib.dptr(g), k, 0.0, _lib.dptr(y),
                                ld_of(y)), reps=5)
    print(f"{'Q R^-1 (zgemm_nn, DMMA)':34s} {ms:8.3f} ms  {8.0 * n * k * k / ms / 1e9:8.2f} TFLOP/s (8 n k^2)")
    rows.append({"kernel": "Q R^-1 (zgemm_nn)", "ms": round(ms, 4), "TFLOP/s": round(8.0 * n * k * k / ms / 1e9, 2),
                 "what": "CholQR update / Ritz back-transform, compute-bound"})
    out_path = Path(__file__).resolve().parents[1] / "gpurun_out" / "hbm_kernels.json"
    out_path.parent.mkdir(exist_ok=True)
    out_path.write_text(json.dumps({"m": m, "n": n, "k": k, "hbm_peak_gbs": PEAK, "kernels": rows}, indent=1))


if __name__ == "__main__":
    main()
