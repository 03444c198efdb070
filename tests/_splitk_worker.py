"""Worker of test_gpu_parity.test_rs_split_k (run in a subprocess: BSE200_RS_KSPLIT is read when the
device context is created).  Prints one JSON line: per shape, the largest difference between the
split-K products (code 98) and the unsplit tile (code 97), relative to the output scale, for the
real-split filter and the grid's transposed-tile product, and whether a repeat is bitwise equal."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_10557_b200 import _lib
from paper_2601_10557_b200.dist import CudaOps, plane_tiles, tile_from_blocks
from paper_2601_10557_b200.hamiltonian import colmajor_empty, ld_of


def main():
    dev = torch.device("cuda", 0)
    ops = CudaOps(dev)
    ctx = ops.ctx
    ctx.set_ham_flags(0)
    gen = torch.Generator(device=dev).manual_seed(17)

    def rnd(*shape):
        return torch.complex(torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64),
                             torch.randn(*shape, generator=gen, device=dev, dtype=torch.float64))

    out = []
    for m, kc, k in ((203, 157, 530), (37, 37, 7), (9, 5, 1), (130, 300, 45)):
        # filter on a square operator's planes (m x m blocks)
        ab = colmajor_empty(m, 2 * m, dev)
        ab.copy_(rnd(m, 2 * m))
        ldg = m + (m & 1)
        gp = torch.empty((4 * m, ldg), dtype=torch.float64, device=dev).t()
        ctx.call("bse_make_rs_planes", _lib.dptr(ab), ld_of(ab), m, m, _lib.dptr(gp), ldg)
        v0 = colmajor_empty(2 * m, k, dev)
        v0.copy_(rnd(2 * m, k))
        work = torch.empty(2 * 2 * m * k, dtype=torch.complex128, device=dev)
        filt = {}
        for code in (97, 98, 98):
            ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, code))
            v = v0.clone()
            ctx.call("bse_chebyshev_filter_rs", _lib.dptr(gp), ldg, m, _lib.dptr(v), 2 * m, k, 4, 0.5, 2.0, -3.0,
                     _lib.dptr(work))
            filt.setdefault(code, []).append(v)
        # transposed product of an m x kc tile (shift rows, beta term)
        fwd, trn = plane_tiles(ops, tile_from_blocks(ops, rnd(m, kc), rnd(m, kc)))
        x, p = rnd(k, 2 * m), rnd(k, 2 * kc)
        tr = {}
        for code in (97, 98, 98):
            ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, code))
            y = torch.zeros(k, 2 * kc, dtype=torch.complex128, device=dev)
            ops.hop(trn, x, y, alpha=0.75, shift=3.5, shift_rows=(1, min(m, kc) - 1), s_off=1, beta=0.25, p=p,
                    filter=True, rs=True)
            tr.setdefault(code, []).append(y)
        torch.cuda.synchronize()

        def rel(a, b):
            return float((a - b).abs().max() / b.abs().max())

        out.append({"m": m, "kc": kc, "k": k, "filter_rel": rel(filt[98][0], filt[97][0]),
                    "trans_rel": rel(tr[98][0], tr[97][0]),
                    "repeat_bitwise": bool(torch.equal(filt[98][0], filt[98][1]) and torch.equal(tr[98][0], tr[98][1]))})
    ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, 90))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
