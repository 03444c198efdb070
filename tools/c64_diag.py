"""Accuracy of the tcgen05 c64 filter vs K (= 2m): degree-2 filter against the FP64 oracle,
with numpy complex64 as the FP32 yardstick."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2601_10557_b200 as bse
from oracle import bse_oracle as o

for m in (64, 300, 1000, 2000, 4000):
    rs = np.random.default_rng(m)
    a = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
    a = a @ a.conj().T / m + np.eye(m)
    a = (a + a.conj().T) / 2
    b = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
    b = 0.1 * (b + b.T) / 2
    x = rs.standard_normal((2 * m, 64)) + 1j * rs.standard_normal((2 * m, 64))
    ham = bse.BseHamiltonian(a, b)
    cfg = bse.FilterConfig(2, 1.0, 3.0, -5.0)
    bse.set_filter_precision("c64")
    out = bse.chebyshev_filter(ham, x, cfg)
    bse.set_filter_precision("c128")
    out128 = bse.chebyshev_filter(ham, x, cfg)
    ref = o.cheb_filter(a, b, x, 2, 1.0, 3.0, -5.0)
    c = o.cheb_filter(a.astype(np.complex64), b.astype(np.complex64), x.astype(np.complex64), 2, np.float32(1.0),
                      np.float32(3.0), np.float32(-5.0))
    sc = np.abs(ref).max()
    print(f"m={m} K={2 * m}: tcgen05 c64 rel err {np.abs(out - ref).max() / sc:.3e}   numpy c64 "
          f"{np.abs(c - ref).max() / sc:.3e}   DMMA c128 {np.abs(out128 - ref).max() / sc:.3e}", flush=True)
