"""Where the end-to-end seconds beyond the device-resident solve go at C3 (bench.py's e2e leg):
H2D of the pinned A, B blocks (device_blocks), the real-split planes, the start block, the
result read-back.  Run: python tools/e2e_breakdown.py [m]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2601_10557_b200 as bse
from paper_2601_10557_b200 import BseHamiltonian, Definiteness
from bench import pinned_fortran


def sync_time(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main(m=20000):
    dev = torch.device("cuda", 0)
    ham = bse.generate(bse.GeneratorSpec(m=m, seed=0))
    a_h, b_h = (pinned_fortran(x) for x in ham.host_blocks())
    ham.release_device()
    del ham
    torch.cuda.empty_cache()
    out = {"m": m, "bytes_ab": 2 * a_h.nbytes}
    for rep in range(3):
        h = BseHamiltonian(a_h, b_h, Definiteness.DEFINITE)
        _, t = sync_time(lambda: h.device_blocks(dev))
        out.setdefault("h2d_s", []).append(round(t, 4))
        _, t = sync_time(lambda: h.device_rs_planes(dev, reserve=0))
        out.setdefault("planes_s", []).append(round(t, 4))
        h.release_device()
        del h
        torch.cuda.empty_cache()
    gbps = out["bytes_ab"] / min(out["h2d_s"]) / 1e9
    out["h2d_gbs"] = round(gbps, 1)
    # raw pinned copy of one block for comparison
    buf = torch.empty((m, m), dtype=torch.complex128, device=dev)
    src = torch.from_numpy(a_h.T)  # (m, m) C-contiguous view of the F-ordered block
    _, t = sync_time(lambda: buf.copy_(src))
    out["raw_h2d_one_block_gbs"] = round(a_h.nbytes / t / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20000)
