"""Microbenchmark of the fused H-operator filter step at the C2/C3 shapes
(random A/B, CUDA events on the launching stream)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_10557_b200 import _lib
from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of


def run(m, k, reps=5):
    dev = torch.device("cuda", 0)
    ab = colmajor_empty(m, 2 * m, dev)
    ab.real.normal_()
    ab.imag.normal_()
    n = 2 * m
    y = colmajor_empty(n, k, dev); y.real.normal_(); y.imag.normal_()
    yp = colmajor_empty(n, k, dev); yp.real.normal_(); yp.imag.normal_()
    ctx = _lib.Context.get(0)
    args = lambda: (_lib.dptr(ab), None, ld_of(ab), m, _lib.dptr(y), _lib.dptr(yp), _lib.dptr(yp), n, k, 0.1, 1e-3, 0.5)
    for _ in range(2):
        ctx.call("bse_filter_step", *args())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.call("bse_filter_step", *args())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 8.0 * n * n * k
    print(f"filter step m={m} k={k}: {ms:.2f} ms  {fl / ms / 1e9:.2f} TFLOP/s (model 8n^2k)")
    del ab, y, yp
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for m, k in [(10000, 600), (10000, 113), (20000, 1200), (20000, 200), (4000, 240)]:
        run(m, k)
