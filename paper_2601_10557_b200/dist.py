"""2D block-distributed pseudo-hermitian ChASE over a p x q grid of GPUs.

The scheme of PAPER.md:723-740 (not shipped by the reference):

* GPU (I, J) of a p x q grid (8 -> 2 x 4, 4 -> 2 x 2, 2 -> 1 x 2) owns the
  tiles A[R_I, C_J], B[R_I, C_J] and their block transposes A[C_J, R_I] =
  A[R_I, C_J]^H, B[C_J, R_I] = B[R_I, C_J]^T (A hermitian, B symmetric), i.e.
  only blocks of A and B — 4 m^2 / (p q) x 16 bytes per GPU.
* Vectors live in one of two layouts: "col" (rows C_J of both halves,
  replicated down the column communicator) and "row" (rows R_I, replicated
  along the row communicator).  A forward tile product maps col -> row and is
  summed over the row communicator; the transposed-tile product maps row ->
  col and is summed over the column communicator (the block form of
  H V = W <=> H^* S V = S W).  The filter alternates the two, so an even
  degree returns V to its starting layout without ever moving A or B.
* The Chebyshev shift term -c Y is folded into the partial product on the
  rows where a tile's input and output blocks intersect, the -beta Y_prev
  term is added by one designated member, so the summed partials ARE
  Y_{j+1}: the whole recurrence is one fused DMMA GEMM + one allreduce per
  step, with two buffers (one per layout) and no copies.
* CholQR Grams, the projection against the locked vectors, [W | Q2^H Q2] and
  [column norms | residual norms] are local partial products plus ONE
  allreduce each; the replicas of a layout split the rows between them.  The
  k x k pencil (solved redundantly in PAPER.md:725) is split into its two
  independent halves on ranks 0 and 1.  Q is redistributed once per iteration
  from the col to the row layout (point-to-point inside the row group); the
  backup projection reuses the same T.
* The complex64 filter (configs[4]) runs the same recurrence on the tcgen05
  tile kernel: raw fp32 partials, an fp32 allreduce, then the hi/lo split.

Everything device-side goes through an ``ops`` object: ``CudaOps`` (the bse200
C ABI) in production; the CPU gloo tests substitute a torch reference.
Vectors are held as "storage" tensors of shape (k, rows) (column-major
matrices rows x k, leading dimension = rows), so column slices are contiguous
for the collectives.
"""

from __future__ import annotations

import ctypes
from functools import partial
import logging
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, rng
from .chebyshev import FilterConfig
from .errors import HermitianRqError, LanczosBreakdownError, NumericalError, RankDeficiencyError, ValidationError
from .generate import EXACT_LIMIT
from .lanczos import MAX_RESTARTS, SAFETY_INFLATION, SpectralBounds, _cutoff, update_cutoff
from .metrics import PhaseLedger
from .rayleigh_ritz import lock_converged, RitzSet
from .solver import SolveResult, SolverConfig, TraceRecord, TAG_LANCZOS, TAG_SUBSPACE

ZB = 16  # bytes per complex128
_TIMING = __import__("os").environ.get("BSE200_TIMING") == "1"


logger = logging.getLogger("paper_2601_10557_b200.dist")


class _Steps:
    """Opt-in step timer (BSE200_TIMING=1): device-synchronised wall time per step on rank 0."""

    def __init__(self, name, rank):
        self.name, self.on = name, _TIMING and rank == 0
        if self.on:
            import time
            import torch

            self.torch, self.time = torch, time
            torch.cuda.synchronize()
            self.t = time.perf_counter()

    def mark(self, step, k=-1):
        if self.on:
            self.torch.cuda.synchronize()
            t = self.time.perf_counter()
            print(f"[dist {self.name} k={k}] {step:<24s} {1e3 * (t - self.t):8.2f} ms", flush=True)
            self.t = t


def grid_shape(world: int) -> tuple[int, int]:
    """Grid as square as possible with p <= q."""
    p = int(math.isqrt(world))
    while world % p:
        p -= 1
    return p, world // p


def split(m: int, parts: int) -> list[int]:
    base, extra = divmod(m, parts)
    edges = [0]
    for i in range(parts):
        edges.append(edges[-1] + base + (1 if i < extra else 0))
    return edges


class Grid:
    """Block ownership of the m x m index space on a p x q grid."""

    def __init__(self, m: int, world: int, rank: int, p: int | None = None, q: int | None = None):
        if p is None or q is None:
            p, q = grid_shape(world)
        if p * q != world:
            raise ValidationError(f"grid {p}x{q} does not match world size {world}")
        self.m, self.p, self.q, self.world, self.rank = m, p, q, world, rank
        self.I, self.J = divmod(rank, q)
        self.re, self.ce = split(m, p), split(m, q)
        self.r0, self.r1 = self.re[self.I], self.re[self.I + 1]
        self.c0, self.c1 = self.ce[self.J], self.ce[self.J + 1]
        self.nr, self.nc = self.r1 - self.r0, self.c1 - self.c0
        # rows shared by the output and input blocks of a forward (col -> row) product,
        # in output-row coordinates; the transposed product uses the same global interval
        lo, hi = max(self.r0, self.c0), min(self.r1, self.c1)
        self.diag = (lo, hi) if hi > lo else (0, 0)

    def row_members(self) -> list[int]:
        return [self.I * self.q + j for j in range(self.q)]

    def col_members(self) -> list[int]:
        return [i * self.q + self.J for i in range(self.p)]


class Comm:
    """Row / column communicators of the grid (torch.distributed groups; NCCL on GPUs, gloo in tests)."""

    def __init__(self, grid: Grid):
        self.g = grid
        self.row = self.col = None
        if grid.world > 1:
            import torch.distributed as dist

            self.dist = dist
            rows = [dist.new_group([i * grid.q + j for j in range(grid.q)]) for i in range(grid.p)]
            cols = [dist.new_group([i * grid.q + j for i in range(grid.p)]) for j in range(grid.q)]
            self.row, self.col = rows[grid.I], cols[grid.J]

    @staticmethod
    def _real(t):
        import torch

        return torch.view_as_real(t) if t.is_complex() else t

    def sum_row(self, t) -> None:
        if self.g.q > 1:
            self.dist.all_reduce(self._real(t), group=self.row)

    def sum_col(self, t) -> None:
        if self.g.p > 1:
            self.dist.all_reduce(self._real(t), group=self.col)

    def sum_all(self, t) -> None:
        if self.g.world > 1:
            self.dist.all_reduce(self._real(t))

    def bcast_all(self, t, src: int) -> None:
        if self.g.world > 1:
            self.dist.broadcast(self._real(t), src=src)

    def max_all(self, t) -> None:
        if self.g.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)

    def min_all(self, t) -> None:
        if self.g.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)

    def gather(self, t, group: str) -> list:
        """allgather of equally shaped contiguous tensors within the row / col group."""
        import torch

        size = self.g.q if group == "row" else self.g.p
        if size == 1:
            return [t]
        outs = [torch.empty_like(t) for _ in range(size)]
        self.dist.all_gather([self._real(o) for o in outs], self._real(t), group=self.row if group == "row" else self.col)
        return outs


# ----------------------------------------------------------------------------- device ops (C ABI)
class CudaOps:
    """Thin wrappers over the bse200 C ABI for the distributed algorithm."""

    def __init__(self, device):
        import torch

        self.torch = torch
        self.device = device
        self.ctx = _lib.Context.get(device.index)

    def empty(self, k: int, rows: int):
        return self.torch.empty((k, rows), dtype=self.torch.complex128, device=self.device)

    def hop(self, tile, x, y, *, alpha=1.0, shift=0.0, shift_col=None, shift_rows=(0, 0), s_off=0, beta=0.0,
            p=None, low_sign=1.0, filter=False, rs=False):
        """y (storage k x 2 mr) = low_sign^{low} (alpha (tile-product of x - shift s) - beta p).
        rs: x, y, s and p are folded (X1 + X2, X1 - X2) and the product runs on the tile's
        real-split planes (bse_hop_tile_rs)."""
        k = x.shape[0]
        mr, kc = tile.mr, tile.kc
        xa, ya = x.data_ptr(), y.data_ptr()
        args = _lib.HopTileArgs()
        args.pa, args.pb, args.lda, args.mr, args.kc = tile.pa, tile.pb, tile.lda, mr, kc
        if filter and tile.sd is not None:
            args.sa, args.sb = tile.sa, tile.sb
        args.x1, args.x2, args.ldx, args.k = xa, xa + kc * ZB, x.stride(0), k
        args.y1, args.y2, args.ldy = ya, ya + mr * ZB, y.stride(0)
        lo, hi = shift_rows
        if (shift != 0.0 or shift_col is not None) and hi > lo:
            args.s1, args.s2, args.lds = xa + s_off * ZB, xa + (kc + s_off) * ZB, x.stride(0)
            args.shift_lo, args.shift_hi = lo, hi
            args.shift = shift
            args.d_shift_col = shift_col.data_ptr() if shift_col is not None else None
        if beta != 0.0:
            pa_ = p.data_ptr()
            args.p1, args.p2, args.ldp = pa_, pa_ + mr * ZB, p.stride(0)
        args.alpha, args.beta, args.low_sign = alpha, beta, low_sign
        args.filter = 1 if filter else 0
        if rs:
            self.ctx.call("bse_hop_tile_rs_t" if tile.trans else "bse_hop_tile_rs", ctypes.byref(args),
                          tile.g.data_ptr(), tile.ldg)
        else:
            self.ctx.call("bse_hop_tile", ctypes.byref(args))

    def make_rs_planes(self, tile):
        """Real-split planes [Z | V | U | W] (mr x 4kc doubles, leading dim ldg) of a complex tile."""
        ldg = tile.mr + (tile.mr & 1)
        g = self.torch.empty((4 * tile.kc, ldg), dtype=self.torch.float64, device=self.device)
        self.ctx.call("bse_make_rs_planes", tile.buf.data_ptr(), tile.lda, tile.mr, tile.kc, g.data_ptr(), ldg)
        return g, ldg

    def rs_fold(self, v, rows: int, scale: float, scale2: float | None = None, out=None):
        """(X1, X2) -> (scale (X1 + X2), scale2 (X1 - X2)) of a (k x 2 rows) storage block into out
        (default: in place; same strides), bse_rs_fold."""
        out = v if out is None else out
        self.ctx.call("bse_rs_fold", v.data_ptr(), out.data_ptr(), v.stride(0), rows, v.shape[0], scale,
                      scale if scale2 is None else scale2)

    # ---- complex64 filter (tcgen05, c64.cuh): plane sets of 8 fp32 planes ----------------------
    @staticmethod
    def _pad4(rows: int) -> int:
        return (rows + 3) // 4 * 4

    def c64_planes(self, rows: int, k: int):
        """Plane set of a (k, 2 rows) block: 8 x 2 pad4(rows) k fp32."""
        return self.torch.empty(8 * 2 * self._pad4(rows) * k, dtype=self.torch.float32, device=self.device)

    def c64_raw(self, rows: int, k: int):
        """Unsplit fp32 (Re, Im) planes of a (k, 2 rows) block, the allreduce payload."""
        return self.torch.empty(2 * 2 * self._pad4(rows) * k, dtype=self.torch.float32, device=self.device)

    def c64_raw_view(self, raw, rows: int, k: int):
        return raw[:2 * 2 * self._pad4(rows) * k]

    def c64_tile_planes(self, tile, src):
        """P planes of `tile` (mo = tile.mr, kc = tile.kc) from the columns of its transposed tile."""
        pl = self.torch.empty(4 * tile.mr * 2 * self._pad4(tile.kc), dtype=self.torch.float32, device=self.device)
        self.ctx.call("bse_c64_tile_planes", src.pa, src.pb, src.lda, tile.mr, tile.kc, pl.data_ptr())
        return pl

    def c64_to_planes(self, v, rows: int, planes):
        self.ctx.call("bse_c64_to_planes", v.data_ptr(), v.stride(0), rows, v.shape[0], planes.data_ptr())

    def c64_from_planes(self, planes, rows: int, v):
        self.ctx.call("bse_c64_from_planes", planes.data_ptr(), rows, v.shape[0], v.data_ptr(), v.stride(0))

    def c64_step(self, pplanes, tile, k: int, x, out, *, alpha, shift, shift_rows, s_off, beta=0.0, prev=None):
        """raw out = alpha (tile product of x - shift x on shift_rows) - beta prev (unsplit fp32)."""
        a = _lib.C64TileArgs()
        a.pplanes, a.mo, a.kc, a.k = pplanes.data_ptr(), tile.mr, tile.kc, k
        a.x, a.out = x.data_ptr(), out.data_ptr()
        a.prev = prev.data_ptr() if (prev is not None and beta != 0.0) else None
        a.alpha, a.beta, a.shift = alpha, beta, shift
        lo, hi = shift_rows
        a.shift_lo, a.shift_hi, a.s_off = (lo, hi, s_off) if hi > lo else (0, 0, 0)
        a.raw = 1
        self.ctx.call("bse_c64_tile_step", ctypes.byref(a))

    def c64_split(self, raw, rows: int, k: int, planes):
        self.ctx.call("bse_c64_split", raw.data_ptr(), rows, k, planes.data_ptr())

    def gram(self, a, b):
        """a^H b for storage blocks with equal rows -> (k2, k1) storage of the k1 x k2 result."""
        k1, rows = a.shape
        k2 = b.shape[0]
        out = self.empty(k2, k1)
        self.ctx.call("bse_zgemm_cn", k1, k2, rows, 1.0, _lib.dptr(a), a.stride(0), _lib.dptr(b), b.stride(0), 0.0,
                      _lib.dptr(out), k1)
        return out

    def nn(self, a, w, out=None, alpha=1.0, beta=0.0):
        """out = alpha a @ W + beta out ; a storage (k1, rows), w storage (k2, k1) of a k1 x k2 matrix."""
        k1, rows = a.shape
        k2 = w.shape[0]
        if out is None:
            out = self.empty(k2, rows)
        self.ctx.call("bse_zgemm_nn", rows, k2, k1, alpha, _lib.dptr(a), a.stride(0), _lib.dptr(w), w.stride(0),
                      beta, _lib.dptr(out), out.stride(0))
        return out

    def chol_rinv(self, g, shift=0.0, rdiag=None):
        k = g.shape[0]
        rinv = self.empty(k, k)
        info = ctypes.c_int(0)
        self.ctx.call("bse_chol_rinv", _lib.dptr(g), k, shift, _lib.dptr(rinv),
                      _lib.dptr(rdiag) if rdiag is not None else None, ctypes.byref(info))
        return rinv, info.value

    def rr_pencil(self, w, g2):
        k = w.shape[0]
        lam = np.zeros(k)
        wvec = self.empty(k, k)
        lmm = ctypes.c_double(0.0)
        self.ctx.call("bse_rr_pencil", _lib.dptr(w), _lib.dptr(g2), k, _lib.hptr(lam), _lib.dptr(wvec),
                      ctypes.byref(lmm))
        return lam, wvec, lmm.value

    def rr_pencil_part(self, part, w, g2):
        """bse_rr_pencil_part: part 1 -> |lambda|_min(M); part 2 -> (lam, wvec) without M's spectrum."""
        k = w.shape[0]
        lam = np.zeros(k)
        wvec = self.empty(k, k)
        lmm = ctypes.c_double(0.0)
        self.ctx.call("bse_rr_pencil_part", part, _lib.dptr(w), _lib.dptr(g2), k, _lib.hptr(lam), _lib.dptr(wvec),
                      ctypes.byref(lmm))
        return lmm.value if part == 1 else (lam, wvec)

    def rr_backup_pencil(self, g0, w, g2):
        k = w.shape[0]
        lam = np.zeros(k)
        y = self.empty(k, k)
        lmm = ctypes.c_double(0.0)
        self.ctx.call("bse_rr_backup_pencil", _lib.dptr(g0), _lib.dptr(w), _lib.dptr(g2), k, _lib.hptr(lam),
                      _lib.dptr(y), ctypes.byref(lmm))
        return lam, y, lmm.value

    def colnorm2(self, x):
        out = self.torch.empty(x.shape[0], dtype=self.torch.float64, device=self.device)
        self.ctx.call("bse_colnorm2", _lib.dptr(x), x.shape[1], x.shape[0], x.stride(0), _lib.dptr(out))
        return out

    def colscale_rsqrt(self, x, n2):
        self.ctx.call("bse_colscale_rsqrt", _lib.dptr(x), x.shape[1], x.shape[0], x.stride(0), _lib.dptr(n2))

    def resid_partial(self, u, v, half, uscale, lam):
        """out[j] = sum_i |sgn_i u_ij uscale_j - lam_j v_ij|^2 (sgn = -1 on rows >= half)."""
        k = u.shape[0]
        out = self.torch.empty(k, dtype=self.torch.float64, device=self.device)
        self.ctx.call("bse_resid_partial", _lib.dptr(u), u.stride(0), _lib.dptr(v), v.stride(0), u.shape[1], half, k,
                      _lib.dptr(uscale), _lib.dptr(lam), _lib.dptr(out))
        return out

    def defect(self, g) -> float:
        out = ctypes.c_double(0.0)
        self.ctx.call("bse_defect", _lib.dptr(g), g.shape[0], ctypes.byref(out))
        return out.value

    def sflip(self, x):
        y = self.empty(x.shape[0], x.shape[1])
        self.ctx.call("bse_sflip", _lib.dptr(x), x.stride(0), _lib.dptr(y), y.stride(0), x.shape[1] // 2, x.shape[0])
        return y


@dataclass
class Tile:
    """[P_A | P_B] of one tile product: pa, pb device addresses, mr x kc each, leading dim lda;
    sd: optional 3M sum planes of the same tile (sa, sb addresses)."""

    buf: object
    pa: int
    pb: int
    lda: int
    mr: int
    kc: int
    sd: object = None
    sa: int = 0
    sb: int = 0
    g: object = None  # optional real-split planes (csrc/hop_rs.cuh), mr x 4kc doubles, leading dim ldg
    ldg: int = 0
    trans: bool = False  # the block transpose of the tile whose planes g holds (bse_hop_tile_rs_t)


def plane_tiles(ops, tile: Tile) -> tuple[Tile, Tile]:
    """(forward, transposed) views of ONE set of real-split planes built from the complex tile
    (A, B)[R_I, C_J]; the complex tile can be freed afterwards.  The transposed view computes the
    row -> col product with A[C_J, R_I] = A[R_I, C_J]^H, B[C_J, R_I] = B[R_I, C_J]^T read from the
    same planes (hop_rs.cuh), so this is the whole operator storage of a grid GPU: 32 mr kc bytes."""
    g, ldg = ops.make_rs_planes(tile)
    fwd = Tile(None, 0, 0, 0, tile.mr, tile.kc, g=g, ldg=ldg)
    trn = Tile(None, 0, 0, 0, tile.kc, tile.mr, g=g, ldg=ldg, trans=True)
    return fwd, trn


def complex_tiles_from_planes(ops, fwd: Tile) -> tuple[Tile, Tile]:
    """Complex (A_t | B_t) forward and transposed tiles rebuilt from the planes (Ar = (V + U)/2,
    Br = (U - V)/2, Ai = (Z + W)/2, Bi = (Z - W)/2; exact to rounding), for the complex64 filter's
    plane conversion only (a temporary; FP32 accuracy there)."""
    torch = ops.torch
    mr, kc = fwd.mr, fwd.kc
    gm = fwd.g.t()[:mr]  # (mr, 4 kc) view, column-major
    z, v, u, w = (gm[:, q * kc:(q + 1) * kc] for q in range(4))
    a_t = torch.complex((v + u) * 0.5, (z + w) * 0.5)
    b_t = torch.complex((u - v) * 0.5, (z - w) * 0.5)
    out = []
    for at, bt in ((a_t, b_t), (a_t.conj().T, b_t.T)):
        rows, cols = at.shape
        buf = torch.empty((2 * cols, rows), dtype=torch.complex128, device=ops.device)
        buf[:cols].copy_(at.T)
        buf[cols:].copy_(bt.T)
        addr = buf.data_ptr()
        out.append(Tile(buf, addr, addr + rows * cols * ZB, rows, rows, cols))
    return tuple(out)


def add_sum_planes(ops, tile: Tile, reserve: int = 0) -> Tile:
    """Attach the 3M (re+im, re-im) planes of the tile (CUDA ops only), if they leave `reserve` bytes
    of HBM for the solve; else the tile product forms the operand sums in registers."""
    if not hasattr(ops, "ctx"):
        return tile
    if not _lib.planes_fit(tile.buf.numel() * 16, ops.device, reserve):
        logger.warning("3M sum planes of a %d x %d tile do not fit; forming the operand sums in registers",
                       tile.mr, 2 * tile.kc)
        return tile
    sd = ops.torch.empty_like(tile.buf)
    ops.ctx.call("bse_make_sum_planes", tile.buf.data_ptr(), tile.lda, tile.mr, 2 * tile.kc, sd.data_ptr())
    tile.sd, tile.sa = sd, sd.data_ptr()
    tile.sb = tile.sa + tile.mr * tile.kc * ZB
    return tile


def tile_from_blocks(ops, a_t, b_t, transpose: bool = False) -> Tile:
    """One column-major [A_t | B_t] device buffer from tile blocks (host numpy or device tensors);
    transpose: the block transpose [A_t^H | B_t^T] instead."""
    torch = ops.torch
    if transpose:
        a_t = a_t.conj().T
        b_t = b_t.T
    mr, kc = a_t.shape
    buf = torch.empty((2 * kc, mr), dtype=torch.complex128, device=ops.device)  # storage of mr x 2kc
    for h, blk in enumerate((a_t, b_t)):
        src = torch.from_numpy(np.ascontiguousarray(blk.T)) if isinstance(blk, np.ndarray) else blk.T
        buf[h * kc:(h + 1) * kc].copy_(src)
    addr = buf.data_ptr()
    return Tile(buf, addr, addr + mr * kc * ZB, mr, mr, kc)


def slice_tile(ops, rows, cols, a_blocks, b_blocks) -> Tile:
    """The tile (A, B)[rows, cols] of full (host or device) blocks."""
    (r0, r1), (c0, c1) = rows, cols
    return tile_from_blocks(ops, a_blocks[r0:r1, c0:c1], b_blocks[r0:r1, c0:c1])


# ----------------------------------------------------------------------------- distributed solver
class DistSolver:
    """SPMD solve on one rank of the grid; every rank calls it with the same config."""

    # filter column chunking (allreduce overlapped with the next chunk's GEMM) from this block width
    # on.  Off by default: at C3 the allreduces are ~1-2% of a step and two half-width GEMMs lose
    # more (4 GPUs: filter 13.0 s chunked vs 12.5 s with the first kernels, 10.97 s vs 10.74 s with the
    # TMA kernel, profiles/r01/); BSE200_CHUNK_MIN enables it.
    CHUNK_MIN = int(__import__("os").environ.get("BSE200_CHUNK_MIN", str(1 << 30)))
    # the start block is drawn (and the first filter run) in two column halves from this width on
    START_SPLIT_MIN = 64

    def __init__(self, grid: Grid, comm: Comm, ops, fwd: Tile, trn: Tile):
        self.g, self.c, self.ops, self.fwd, self.trn = grid, comm, ops, fwd, trn
        self.torch = ops.torch
        # real-split mode: this rank stores ONE tile's planes; every product runs on them
        self.planes = fwd.g is not None and trn.g is not None

    # ---- layout helpers -----------------------------------------------------------------
    def col_rows(self, full_storage):
        """col layout [X1[C_J]; X2[C_J]] of a full (k, n) storage block."""
        g, m = self.g, self.g.m
        return self.torch.cat([full_storage[:, g.c0:g.c1], full_storage[:, m + g.c0:m + g.c1]], dim=1).contiguous()

    def assemble_from_col(self, local):
        """allgather the col-layout blocks along the row communicator -> full (k, n) storage."""
        g, torch = self.g, self.torch
        k = local.shape[0]
        mx = max(g.ce[j + 1] - g.ce[j] for j in range(g.q))
        pad = torch.zeros((k, 2 * mx), dtype=local.dtype, device=local.device)
        pad[:, :g.nc] = local[:, :g.nc]
        pad[:, mx:mx + g.nc] = local[:, g.nc:]
        parts = self.c.gather(pad, "row")
        full = torch.empty((k, 2 * g.m), dtype=local.dtype, device=local.device)
        for j, part in enumerate(parts):
            a, b = g.ce[j], g.ce[j + 1]
            full[:, a:b] = part[:, :b - a]
            full[:, g.m + a:g.m + b] = part[:, mx:mx + b - a]
        return full

    def assemble_from_row(self, local):
        """allgather the row-layout blocks along the column communicator -> full (k, n) storage."""
        g, torch = self.g, self.torch
        k = local.shape[0]
        mx = max(g.re[i + 1] - g.re[i] for i in range(g.p))
        pad = torch.zeros((k, 2 * mx), dtype=local.dtype, device=local.device)
        pad[:, :g.nr] = local[:, :g.nr]
        pad[:, mx:mx + g.nr] = local[:, g.nr:]
        parts = self.c.gather(pad, "col")
        full = torch.empty((k, 2 * g.m), dtype=local.dtype, device=local.device)
        for i, part in enumerate(parts):
            a, b = g.re[i], g.re[i + 1]
            full[:, a:b] = part[:, :b - a]
            full[:, g.m + a:g.m + b] = part[:, mx:mx + b - a]
        return full

    def col_to_row(self, x_col):
        """Redistribute a col-layout block (rows C_J of both halves) to the row layout (rows R_I) --
        ChASE's row/column redistribution: inside the row group, member j owns the
        piece C_j ∩ R_I and sends it to the others by point-to-point NCCL, so each GPU receives
        (m/p - |C_J ∩ R_I|) rows of each half instead of allgathering all m."""
        g, torch = self.g, self.torch
        k = x_col.shape[0]
        out = torch.empty((k, 2 * g.nr), dtype=x_col.dtype, device=x_col.device)

        def piece(j):  # C_j ∩ R_I in global rows
            return max(g.ce[j], g.r0), min(g.ce[j + 1], g.r1)

        lo, hi = piece(g.J)
        mine = None
        if hi > lo:  # my own piece: local copy, packed [upper | lower] for the sends
            mine = torch.cat([x_col[:, lo - g.c0:hi - g.c0], x_col[:, g.nc + lo - g.c0:g.nc + hi - g.c0]], dim=1)
            out[:, lo - g.r0:hi - g.r0] = mine[:, :hi - lo]
            out[:, g.nr + lo - g.r0:g.nr + hi - g.r0] = mine[:, hi - lo:]
        if g.q == 1:
            return out
        dist = self.c.dist
        # gloo has no point-to-point transport for CUDA tensors (the 8-ranks-on-4-GPUs test mode):
        # stage those through host memory
        staged = x_col.is_cuda and dist.get_backend() == "gloo"
        dev = torch.device("cpu") if staged else x_col.device
        send = mine.cpu() if (staged and mine is not None) else mine
        ops, recvs = [], []
        for j in range(g.q):
            if j == g.J:
                continue
            peer = g.I * g.q + j
            if send is not None:
                ops.append(dist.P2POp(dist.isend, self.c._real(send), peer))
            plo, phi = piece(j)
            if phi > plo:
                buf = torch.empty((k, 2 * (phi - plo)), dtype=x_col.dtype, device=dev)
                ops.append(dist.P2POp(dist.irecv, self.c._real(buf), peer))
                recvs.append((plo, phi, buf))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for plo, phi, buf in recvs:
            buf = buf.to(x_col.device)
            out[:, plo - g.r0:phi - g.r0] = buf[:, :phi - plo]
            out[:, g.nr + plo - g.r0:g.nr + phi - g.r0] = buf[:, phi - plo:]
        return out

    def row_rows(self, full_storage):
        g, m = self.g, self.g.m
        return self.torch.cat([full_storage[:, g.r0:g.r1], full_storage[:, m + g.r0:m + g.r1]], dim=1).contiguous()

    # ---- H products -----------------------------------------------------------------------
    def forward(self, x_col, y_row, **kw):
        """col -> row partial product, summed over the row communicator into y_row."""
        g = self.g
        lo, hi = g.diag
        hop = partial(self.ops.hop, self.fwd, x_col, y_row, shift_rows=(lo - g.r0, hi - g.r0), s_off=g.r0 - g.c0,
                      **kw)
        if not self._fused_reduce("row", hop, y_row, kw):
            hop()
            self.c.sum_row(y_row)

    def transposed(self, x_row, y_col, **kw):
        """row -> col partial product (block-transposed tiles), summed over the column communicator."""
        g = self.g
        lo, hi = g.diag
        hop = partial(self.ops.hop, self.trn, x_row, y_col, shift_rows=(lo - g.c0, hi - g.c0), s_off=g.c0 - g.r0,
                      **kw)
        if not self._fused_reduce("col", hop, y_col, kw):
            hop()
            self.c.sum_col(y_col)

    # ---- fused tile product + group reduction over NVLink peer memory (BSE200_FUSED_REDUCE=1) -----
    FUSED_REDUCE = __import__("os").environ.get("BSE200_FUSED_REDUCE", "0") == "1"

    def _fused_reduce(self, group: str, hop, y, kw) -> bool:
        """The tile product followed by the group allreduce as ONE real-split kernel whose epilogue
        stores each output tile into this rank's slot of every group member's symmetric inbox
        (NVLink stores, overlapping the transfer with the product tile by tile), a barrier among
        the group, and a local fixed-order sum of the slots (bse_set_push_targets, bse_group_sum).
        Real-split products on CUDA ops under NCCL only; False -> the caller runs hop + allreduce."""
        size = self.g.q if group == "row" else self.g.p
        if not (self.FUSED_REDUCE and size > 1 and size <= 4 and kw.get("rs") and hasattr(self.ops, "ctx")
                and self.c.dist.get_backend() == "nccl" and y.is_contiguous()):
            return False
        k = y.shape[0]
        t, h, cap, ptrs = self._inbox(group, y.shape[1], k)
        ctx = self.ops.ctx
        me = h.rank
        targets = (ctypes.c_void_p * size)(*[ptrs[j] + me * cap * ZB for j in range(size)])
        h.barrier(channel=0, timeout_ms=120000)  # every member has summed its inbox from this group's previous product
        ctx.call("bse_set_push_targets", targets, size)
        try:
            hop()
        finally:
            ctx.call("bse_set_push_targets", None, 0)
        h.barrier(channel=0, timeout_ms=120000)  # every member's stores into this inbox are complete
        ctx.call("bse_group_sum", t.data_ptr(), cap, size, y.data_ptr(), y.numel())
        return True

    def _inbox(self, group: str, width: int, k: int):
        """This rank's symmetric inbox for the group: one slot of >= k x width complex per member."""
        cache = self.__dict__.setdefault("_inboxes", {})
        need = k * width
        ent = cache.get(group)
        if ent is None or ent[2] < need:
            import torch.distributed._symmetric_memory as symm

            size = self.g.q if group == "row" else self.g.p
            pg = self.c.row if group == "row" else self.c.col
            cap = max(need, ent[2] if ent else 0)
            if ent is not None:
                # no kernel of this rank may still read the old inbox, and no peer writes into it
                # outside a product bracketed by the group's barriers: drain, then free
                self.torch.cuda.synchronize(self.ops.device)
                ent[1].barrier(channel=0, timeout_ms=120000)
                self.torch.cuda.synchronize(self.ops.device)
            cache.pop(group, None)
            ent = None
            t = symm.empty(2 * size * cap, dtype=self.torch.float64, device=self.ops.device)
            h = symm.rendezvous(t, pg)
            ent = (t, h, cap, list(h.buffer_ptrs))
            cache[group] = ent
        return ent

    def chebyshev(self, v_col, cfg: FilterConfig, row_buf):
        """p(H) v in place (col layout); row_buf: (k, 2 nr) scratch.  chebyshev.py:58-74.

        H acts on each column independently, so the block is split into column chunks that run
        through the recurrence as independent pipelines: while one chunk's partial product is
        being allreduced (NCCL on a communication stream), the next chunk's tile GEMM runs."""
        c, e = cfg.center, cfg.half_width
        s1 = e / (cfg.scale_ref - c)
        k = v_col.shape[0]
        nch = 1 if (self.g.world == 1 or k < self.CHUNK_MIN) else 2
        edges = split(k, nch)
        torch = self.torch
        overlap = nch > 1 and hasattr(self.ops, "ctx")  # streams only with the CUDA ops
        comp = torch.cuda.current_stream() if overlap else None
        if overlap and not hasattr(self, "_comm_stream"):
            self._comm_stream = torch.cuda.Stream(device=v_col.device)
        reduced = [None] * nch
        # real-split planes: run the recurrence in the folded basis (csrc/hop_rs.cuh)
        rs = self.planes
        if rs:
            self.ops.rs_fold(v_col, self.g.nc, 1.0)
        for ci in range(nch):
            a, b = edges[ci], edges[ci + 1]
            src, dst = v_col[a:b], row_buf[a:b]
            s = s1
            for step in range(1, cfg.degree + 1):
                if step == 1:
                    kw = dict(alpha=s1 / e, shift=c)
                else:
                    sn = 1.0 / (2.0 / s1 - s)
                    owner = self._beta_owner(step)
                    # Y_{j+1} = (2 sn / e)(H Y_j - c Y_j) - (s sn) Y_{j-1}; Y_{j-1} lives in dst (in place)
                    kw = dict(alpha=2.0 * sn / e, shift=c, beta=(s * sn) if owner else 0.0,
                              p=dst if owner else None)
                    s = sn
                if rs:
                    kw["rs"] = True
                fwd = step % 2 == 1
                if overlap:
                    reduced[ci] = self._step_async(src, dst, fwd, kw, comp, reduced[ci])
                else:
                    (self.forward if fwd else self.transposed)(src, dst, filter=True, **kw)
                src, dst = dst, src
        if overlap:
            for ev in reduced:
                comp.wait_event(ev)
        if rs:
            self.ops.rs_fold(v_col, self.g.nc, 0.5)
        return v_col  # even degree: the result is back in the col buffer

    def chebyshev_c64(self, v_col, cfg: FilterConfig):
        """p(H) v in place (col layout) with the complex64 tcgen05 filter (c64.cuh) on the 2D grid.
        Each step: the tile product writes unsplit fp32 partials (the -beta Y_prev term on the
        reduction group's owner, the shift on the rows the tile's input and output blocks share),
        one fp32 allreduce over the row / column communicator, then the split into the hi/lo
        planes the next step's TMA boxes read.  chebyshev.py:58-74, as chebyshev() above."""
        g = self.g
        ops = self.ops
        k = v_col.shape[0]
        if not hasattr(self, "_c64_pl"):
            fwd, trn = complex_tiles_from_planes(ops, self.fwd) if self.planes else (self.fwd, self.trn)
            self._c64_pl = (ops.c64_tile_planes(fwd, trn), ops.c64_tile_planes(trn, fwd))
            del fwd, trn
        pl_fwd, pl_trn = self._c64_pl
        col, row = ops.c64_planes(g.nc, k), ops.c64_planes(g.nr, k)
        raw = ops.c64_raw(max(g.nr, g.nc), k)
        ops.c64_to_planes(v_col, g.nc, col)
        lo, hi = g.diag
        c, e = cfg.center, cfg.half_width
        s1 = e / (cfg.scale_ref - c)
        s = s1
        for step in range(1, cfg.degree + 1):
            fwd = step % 2 == 1
            if step == 1:
                alpha, beta = s1 / e, 0.0
            else:
                sn = 1.0 / (2.0 / s1 - s)
                alpha, beta = 2.0 * sn / e, (s * sn) if self._beta_owner(step) else 0.0
                s = sn
            if fwd:  # col -> row: rows R_I, contraction over C_J, summed over the row communicator
                tile, pl, x, out, rows = self.fwd, pl_fwd, col, row, g.nr
                shift_rows, s_off, reduce = (lo - g.r0, hi - g.r0), g.r0 - g.c0, self.c.sum_row
            else:
                tile, pl, x, out, rows = self.trn, pl_trn, row, col, g.nc
                shift_rows, s_off, reduce = (lo - g.c0, hi - g.c0), g.c0 - g.r0, self.c.sum_col
            ops.c64_step(pl, tile, k, x, raw, alpha=alpha, shift=c, shift_rows=shift_rows, s_off=s_off, beta=beta,
                         prev=out if beta != 0.0 else None)
            reduce(ops.c64_raw_view(raw, rows, k))
            ops.c64_split(raw, rows, k, out)
        ops.c64_from_planes(col, g.nc, v_col)  # even degree: back in the col layout
        return v_col

    def _step_async(self, src, dst, fwd, kw, comp, prev_event):
        """One chunk step: tile GEMM on the compute stream (after the chunk's previous reduction),
        allreduce on the communication stream; returns the event marking the reduced chunk."""
        torch = self.torch
        g = self.g
        if prev_event is not None:
            comp.wait_event(prev_event)
        lo, hi = g.diag
        if fwd:
            self.ops.hop(self.fwd, src, dst, shift_rows=(lo - g.r0, hi - g.r0), s_off=g.r0 - g.c0, filter=True, **kw)
        else:
            self.ops.hop(self.trn, src, dst, shift_rows=(lo - g.c0, hi - g.c0), s_off=g.c0 - g.r0, filter=True, **kw)
        done = torch.cuda.Event()
        done.record(comp)
        cs = self._comm_stream
        with torch.cuda.stream(cs):
            cs.wait_event(done)
            (self.c.sum_row if fwd else self.c.sum_col)(dst)
            red = torch.cuda.Event()
            red.record(cs)
        # keep dst alive for the communication stream's use
        dst.record_stream(cs)
        return red

    def _beta_owner(self, step: int) -> bool:
        # the -beta Y_prev term is added once per reduction group
        return (self.g.I == 0) if step % 2 == 0 else (self.g.J == 0)

    # ---- replicated layouts ------------------------------------------------------------------
    # A col-layout block is replicated on the p ranks of its column group, a row-layout block on the
    # q ranks of its row group.  Reductions over its rows (Grams, column norms, residual partials)
    # therefore let each replica take one contiguous share of the rows and sum over ALL ranks:
    # 1/p (1/q) of the work for the same single allreduce.
    def _share(self, width: int, layout: str) -> tuple[int, int]:
        parts, idx = (self.g.p, self.g.I) if layout == "col" else (self.g.q, self.g.J)
        e = split(width, parts)
        return e[idx], e[idx + 1]

    def _gram_row(self, a, b=None):
        """a^H b over the rows of col-layout blocks (summed over all their rows, every rank gets it)."""
        lo, hi = self._share(a.shape[1], "col")
        gm = self.ops.gram(a[:, lo:hi], (a if b is None else b)[:, lo:hi])
        self.c.sum_all(gm)
        return gm

    def _colnorm2(self, x, layout: str):
        lo, hi = self._share(x.shape[1], layout)
        n2 = self.ops.colnorm2(x[:, lo:hi])
        self.c.sum_all(n2)
        return n2

    def cholqr(self, q_col):
        """Distributed CholQR2 (+ shifted CholQR3 fallback) of a col-layout block; returns (q, method)."""
        st = _Steps("cholqr", self.g.rank)
        x0 = q_col.clone()
        q = q_col
        ok = True
        for p in range(2):
            gm = self._gram_row(q)
            g2 = gm.clone() if p == 1 else None  # chol_rinv factors in place
            st.mark("gram + allreduce", q.shape[0])
            rinv, info = self.ops.chol_rinv(gm)
            st.mark("chol_rinv", q.shape[0])
            if info != 0:
                ok = False
                break
            q = self.ops.nn(q, rinv)
            st.mark("Q R^-1", q.shape[0])
        # defect max|Q^H Q - I| folded into pass 2 (ortho.py:124): Q^H Q = R^-H G2 R^-1 from the pass's
        # own Gram, k x k work and no third Gram + allreduce
        if ok and self.ops.defect(self.ops.gram(rinv, self.ops.nn(g2, rinv))) <= 1e-8:
            st.mark("defect", q.shape[0])
            return q, "cholqr"
        st.mark("FALLBACK", q.shape[0])
        # shifted CholQR3 on the original block
        n2 = self._colnorm2(x0, "col")
        k = x0.shape[0]
        n = 2 * self.g.m
        shift = 11.0 * (n * k + k * (k + 1)) * 2.0**-53 * float(n2.sum().item())
        rd = self.torch.empty(k, dtype=self.torch.float64, device=x0.device)
        prod = np.ones(k)
        q = x0
        for sh in (shift, 0.0, 0.0):
            rinv, info = self.ops.chol_rinv(self._gram_row(q), shift=sh, rdiag=rd)
            if info != 0 or not shift > 0:
                raise RankDeficiencyError("columns are numerically rank deficient (shifted Cholesky failed)")
            prod *= rd.cpu().numpy()
            q = self.ops.nn(q, rinv)
        if not prod.min() > 1e-10 * prod.max():
            raise RankDeficiencyError(f"columns are numerically rank deficient (diag ratio {prod.min():.3e})")
        if not self.ops.defect(self._gram_row(q)) <= 1e-8:
            raise RankDeficiencyError("orthonormalization failed")
        return q, "shifted_cholqr"

    def extend_sbasis(self, sbasis, l_old: int, y_new) -> None:
        """sbasis[l_old:l_old + c] <- orthonormal completion of span(S Y_new) against sbasis[:l_old]
        (col layout; the single-GPU bse_extend_sbasis: BCGS2 then CholQR of the new block only)."""
        c = y_new.shape[0]
        if not c:
            return
        b = self.ops.sflip(y_new)
        if l_old:
            for _ in range(2):
                proj = self._gram_row(sbasis[:l_old], b)
                self.ops.nn(sbasis[:l_old], proj, out=b, alpha=-1.0, beta=1.0)
        q, _ = self.cholqr(b)
        sbasis[l_old:l_old + c].copy_(q)

    def s_orthonormalize(self, v_col, basis):
        """ortho.py:132-158 distributed: project out span(S Y) -- given by its orthonormal basis,
        grown incrementally as pairs lock -- then CholQR2 (col layout)."""
        st = _Steps("s_ortho", self.g.rank)
        if basis is not None and basis.shape[0]:
            proj = self._gram_row(basis, v_col)  # l x k
            self.ops.nn(basis, proj, out=v_col, alpha=-1.0, beta=1.0)
            st.mark("projection", v_col.shape[0])
        q, method = self.cholqr(v_col)
        self.fix_phases(q)
        st.mark("phase convention", q.shape[0])
        return q, method

    def fix_phases(self, q_col) -> None:
        """ortho.py:70-82 on the grid (the single-GPU phase_fix_kernel's convention): each column is
        scaled by conj(p)/|p|, p its first entry in GLOBAL row order (upper half, then lower) with
        |q| >= 1e-8 max|q|.  Three k-length collectives: max, first index, the entry itself (sent by
        the I = 0 replica of the column group that holds it)."""
        torch, g = self.torch, self.g
        k = q_col.shape[0]
        if k == 0:
            return
        if not hasattr(self, "_gidx") or self._gidx.numel() != 2 * g.nc:
            self._gidx = torch.cat([torch.arange(g.c0, g.c1), g.m + torch.arange(g.c0, g.c1)]).to(
                device=q_col.device, dtype=torch.float64)
        mag = q_col.abs()
        top = mag.amax(dim=1) if mag.shape[1] else torch.zeros(k, dtype=torch.float64, device=q_col.device)
        self.c.max_all(top)
        big = float(2 * g.m)
        hit = mag >= (1e-8 * top)[:, None]
        first = torch.where(hit, self._gidx[None, :], torch.full_like(mag, big)).amin(dim=1) if mag.shape[1] else \
            torch.full((k,), big, dtype=torch.float64, device=q_col.device)
        self.c.min_all(first)
        sel = (self._gidx[None, :] == first[:, None]) & hit
        val = (q_col * sel).sum(dim=1) if g.I == 0 else torch.zeros(k, dtype=q_col.dtype, device=q_col.device)
        self.c.sum_all(val)
        ap = val.abs()
        fac = torch.where(ap > 0, val.conj() / torch.where(ap > 0, ap, torch.ones_like(ap)), torch.ones_like(val))
        q_col *= fac[:, None]

    # ---- Rayleigh-Ritz + residuals ------------------------------------------------------------
    def rayleigh_ritz(self, q_col, row_buf, fused_residuals: bool = False, variant: str = "auto", it: int = 0,
                      ledger: PhaseLedger | None = None):
        """rayleigh_ritz.py:98-179 distributed, with the variant policy of solver.py:162-181.
        Returns (lam, v_col, lambda_min_m, residuals or None, variant used, backup fallback taken).
        One T = S H Q serves both projections: its halves give Q^H S H Q = G_top + G_bot (hermitian W,
        backup G0) and Q^H H Q = G_top - G_bot (backup W), so a fallback costs no second H product.
        fused_residuals: H V = S T y / |Q y| from T (rows R_I), no further H product."""
        k = q_col.shape[0]
        n, nr = 2 * self.g.m, self.g.nr
        st = _Steps("rr", self.g.rank)
        t_row = row_buf[:k]
        if self.planes:
            # T = S H Q on the real-split planes: fold Q, tile product + row allreduce, unfold with the S-flip
            q_f = self.torch.empty_like(q_col)
            self.ops.rs_fold(q_col, self.g.nc, 1.0, out=q_f)
            self.forward(q_f, t_row, filter=True, rs=True)
            self.ops.rs_fold(t_row, nr, 0.5, -0.5)
            del q_f
        else:
            self.forward(q_col, t_row, low_sign=-1.0, filter=True)  # T = S H Q (rows R_I), filter kernel
        st.mark("T = S H Q", k)
        q_rows = self.col_to_row(q_col)
        st.mark("redistribute Q (col -> row layout)", k)
        rlo, rhi = self._share(nr, "row")  # this replica's share of the rows of each half
        clo, chi = self._share(self.g.nc, "col")
        nc = self.g.nc
        # [Q^H T (upper rows) | Q^H T (lower rows) | Q2^H Q2]: three partial Grams, ONE allreduce
        grams = self.torch.stack([self.ops.gram(q_rows[:, rlo:rhi], t_row[:, rlo:rhi]),
                                  self.ops.gram(q_rows[:, nr + rlo:nr + rhi], t_row[:, nr + rlo:nr + rhi]),
                                  self.ops.gram(q_col[:, nc + clo:nc + chi], q_col[:, nc + clo:nc + chi])])
        self.c.sum_all(grams)
        gtb, g2 = grams[:2], grams[2]
        st.mark("Q^H T halves, Q2^H Q2 + one allreduce", k)
        used, fallback, lam = "hermitian", False, None
        if ledger is not None:
            ledger.add_flops("rr", 8.0 * n * n * k)  # apply_h inside RR (hamiltonian.py:148-150)
        if variant != "backup":
            try:
                lam, wvec, lmm = self._pencil(gtb[0] + gtb[1], g2)
                if ledger is not None:
                    ledger.add_flops("rr", 8.0 * n * n * k + 12.0 * n * k * k + 16.0 * k**3)
            except HermitianRqError as exc:
                if variant == "hermitian":
                    raise NumericalError(f"hermitian projection failed at iteration {it} with fallback "
                                         f"disabled: {exc}") from exc
                logger.warning("iteration %d: switching to backup projection (%s)", it, exc)
                fallback = True
                if ledger is not None:  # the reference's build_backup_rq applies H again
                    ledger.add_flops("rr", 8.0 * n * n * k)
        if lam is None:
            used = "backup"
            lam, wvec, lmm = self.ops.rr_backup_pencil(gtb[0] + gtb[1], gtb[0] - gtb[1], g2)
            if ledger is not None:
                ledger.add_flops("rr", 8.0 * n * n * k + 20.0 * n * k * k + 30.0 * k**3)
        st.mark("pencil", k)
        torch = self.torch
        v = self.ops.nn(q_col, wvec)
        # column norms of V (col layout) and, fused, the residual partials |S T w - lam Q w|^2 (row
        # layout): one allreduce of both k-vectors
        red = torch.zeros((2, k), dtype=torch.float64, device=v.device)
        lo, hi = self._share(v.shape[1], "col")
        red[0] = self.ops.colnorm2(v[:, lo:hi])
        if fused_residuals:
            ones = torch.ones(k, dtype=torch.float64, device=v.device)
            lam_d = torch.as_tensor(np.ascontiguousarray(lam), dtype=torch.float64, device=v.device)
            for off, half in ((0, rhi - rlo), (nr, 0)):  # upper share (no sign flip), lower share (S: negated)
                sl = slice(off + rlo, off + rhi)
                if rhi > rlo:
                    red[1] += self.ops.resid_partial(self.ops.nn(t_row[:, sl], wvec),
                                                     self.ops.nn(q_rows[:, sl], wvec), half, ones, lam_d)
        self.c.sum_all(red)
        n2 = red[0].contiguous()
        self.ops.colscale_rsqrt(v, n2)
        res = np.sqrt(red[1].cpu().numpy() / n2.cpu().numpy()) if fused_residuals else None
        st.mark("V = Q w, normalise (+ residuals from S T w), one allreduce", k)
        return lam, v, lmm, res, used, fallback

    _PENCIL_ERRORS = {1: "Cholesky of Q*SHQ failed; S*H is not definite on the subspace",
                      2: "reduced spectrum touches zero; cannot invert"}

    def _pencil(self, w, g2):
        """The k x k pencil of the hermitian RR (rayleigh_ritz.py:113-137).  On one GPU as a whole; on a
        grid its two independent halves run concurrently on ranks 1 (eigenvalues of M) and 0 (chol(W),
        G, eigh(G), back-transform), then one small allreduce and one broadcast share the results.
        Errors keep the reference's order: a singular M first, then the Cholesky / theta ~ 0 failures."""
        g = self.g
        if g.world == 1 or not hasattr(self.ops, "rr_pencil_part"):
            return self.ops.rr_pencil(w, g2.clone())
        torch = self.torch
        k = w.shape[0]
        info = torch.zeros(2, dtype=torch.float64, device=w.device)  # [lambda_min(M), error code]
        lam_d = torch.zeros(k, dtype=torch.float64, device=w.device)
        wvec = self.ops.empty(k, k)
        if g.rank == 1:
            info[0] = self.ops.rr_pencil_part(1, w, g2.clone())
        elif g.rank == 0:
            try:
                lam, wvec = self.ops.rr_pencil_part(2, w, g2.clone())
                lam_d.copy_(torch.from_numpy(lam))
            except HermitianRqError as exc:
                info[1] = 1.0 if "Cholesky" in str(exc) else 2.0
        self.c.sum_all(info)
        lmm, code = float(info[0].item()), int(info[1].item())
        if not lmm >= 1e-8:
            raise HermitianRqError(f"|lambda_min(Q*SQ)| = {lmm:.6e} below 1e-8")
        if code:
            raise HermitianRqError(self._PENCIL_ERRORS[code])
        # [w vectors | lambda] in one broadcast
        pack = torch.empty(k * k + k, dtype=torch.complex128, device=w.device)
        if g.rank == 0:
            pack[:k * k].copy_(wvec.reshape(-1))
            pack[k * k:].copy_(lam_d)
        self.c.bcast_all(pack, src=0)
        wvec = pack[:k * k].view(k, k)
        return pack[k * k:].real.cpu().numpy(), wvec, lmm

    def residuals(self, v_col, lam, row_buf) -> np.ndarray:
        k = v_col.shape[0]
        r_row = row_buf[:k]
        lam_d = self.torch.as_tensor(np.ascontiguousarray(lam), dtype=self.torch.float64, device=v_col.device)
        if self.planes:
            # folded: (R1 + R2, R1 - R2) = H_f v_f - Lambda v_f, and |r_x|^2 + |r_y|^2 = 2 |R|^2
            v_f = self.torch.empty_like(v_col)
            self.ops.rs_fold(v_col, self.g.nc, 1.0, out=v_f)
            self.forward(v_f, r_row, shift_col=lam_d, filter=True, rs=True)
            del v_f
            n2 = self._colnorm2(r_row, "row") * 0.5
        else:
            self.forward(v_col, r_row, shift_col=lam_d)  # R = H V - V Lambda (rows R_I)
            n2 = self._colnorm2(r_row, "row")
        return np.sqrt(n2.cpu().numpy())

    # ---- Lanczos (lanczos.py:53-142) ------------------------------------------------------------
    def matvec_full(self, x_full):
        """H x for a full (1, n) storage vector; returns the full product on every rank."""
        y_row = self.ops.empty(1, 2 * self.g.nr)
        x_col = self.col_rows(x_full)
        if self.planes:  # fold, product on the planes, unfold
            self.ops.rs_fold(x_col, self.g.nc, 1.0)
            self.forward(x_col, y_row, filter=True, rs=True)
            self.ops.rs_fold(y_row, self.g.nr, 0.5)
        else:
            self.forward(x_col, y_row)
        return self.assemble_from_row(y_row)

    def lanczos(self, nevex: int, steps: int, seed: int, ledger: PhaseLedger) -> SpectralBounds:
        torch = self.torch
        n, m = 2 * self.g.m, self.g.m
        sgn = torch.ones(n, dtype=torch.float64, device=self.ops.device)
        sgn[m:] = -1.0

        def sdot(x, y):  # Re vdot(S x, y)
            return float(torch.sum(sgn * (x.real * y.real + x.imag * y.imag)).item())

        def sweep(start):
            hr = self.matvec_full(start)
            ledger.add_flops("lanczos", 8.0 * n * n)
            nrm2 = sdot(hr[0], start[0])
            if not nrm2 > 0:
                from .errors import IndefiniteError

                raise IndefiniteError("start vector has non-positive S*H norm; matrix is not definite")
            sc = math.sqrt(nrm2)
            q, z = start / sc, hr / sc
            q_old = torch.zeros_like(q)
            beta_prev, al, be = 0.0, [], []
            for j in range(steps):
                al.append(sdot(z[0], z[0]))
                if j == steps - 1:
                    break
                w = z - al[-1] * q - beta_prev * q_old
                gv = self.matvec_full(w)
                ledger.add_flops("lanczos", 8.0 * n * n)
                b2 = sdot(gv[0], w[0])
                if b2 <= (1e-14 * max(1.0, max(abs(a) for a in al), beta_prev)) ** 2:
                    break
                beta = math.sqrt(b2)
                be.append(beta)
                q_old, q = q, w / beta
                z = gv / beta
                beta_prev = beta
            return np.array(al), np.array(be), len(al) < steps

        al = be = np.empty(0)
        for attempt in range(MAX_RESTARTS + 1):
            st = torch.from_numpy(rng.complex_normals(rng.substream(seed, attempt), n)).to(self.ops.device)[None, :]
            al, be, early = sweep(st)
            if not early or len(al) >= min(4, steps):
                break
        if len(al) < min(4, steps):
            raise LanczosBreakdownError(f"Lanczos broke down before {min(4, steps)} steps")
        if len(al) % 2:
            al = al[:-1]
            be = be[: len(al) - 1]
        import scipy.linalg as sla

        theta, y = sla.eigh_tridiagonal(al, be)
        wts = y[0, :] ** 2
        mu_1 = float(theta[0]) - SAFETY_INFLATION * abs(float(theta[0]))
        cut = float(min(max(_cutoff(theta, wts, nevex, n), mu_1), -mu_1))
        return SpectralBounds(mu_1=mu_1, mu_nevex=cut, mu_n=-mu_1, steps=len(al), ritz_values=theta,
                              ritz_weights=wts)

    # ---- outer loop (solver.py:125-250) -----------------------------------------------------------
    def solve(self, cfg: SolverConfig) -> SolveResult:
        torch = self.torch
        g = self.g
        n, nevex, nev, tol = 2 * g.m, cfg.nevex, cfg.nev, cfg.tol
        cfg.validate(n)
        if self.FUSED_REDUCE and self.planes and hasattr(self.ops, "ctx") and g.world > 1:
            # the fused reductions' symmetric inboxes at full width up front (collective; no regrowth)
            if g.q > 1:
                self._inbox("row", 2 * g.nr, nevex)
            if g.p > 1:
                self._inbox("col", 2 * g.nc, nevex)
        ledger = PhaseLedger()
        st = _Steps("solve", g.rank)
        seed3 = rng.substream(cfg.seed, TAG_SUBSPACE)
        host_draw = g.m <= EXACT_LIMIT or not hasattr(self.ops, "ctx")
        pool = second = None
        k1 = nevex
        if host_draw:
            # bit-exact host draw in two column halves on a helper thread: the first during the
            # Lanczos sweep, the second during the first half's filter (columns are independent)
            from concurrent.futures import ThreadPoolExecutor

            k1 = nevex // 2 if nevex >= self.START_SPLIT_MIN else nevex
            pool = ThreadPoolExecutor(1)
            first = pool.submit(start_block_host, seed3, n, 0, k1, g, self.c)
            second = pool.submit(start_block_host, seed3, n, k1, nevex, g, self.c) if k1 < nevex else None
        with ledger.timing("lanczos"):
            bounds = self.lanczos(nevex, cfg.lanczos_steps, rng.substream(cfg.seed, TAG_LANCZOS), ledger)
        st.mark("lanczos", nevex)
        normalizer = abs(bounds.mu_1) if cfg.rel_res else 1.0
        if host_draw:
            v = self.ops.empty(nevex, 2 * g.nc)
            v[:k1] = start_block_finish(first.result(), 0, k1, g, self.ops, self.c)
        else:
            v = start_block_col(seed3, n, nevex, g, self.ops, self.c)
        st.mark("start block", nevex)
        row_buf = self.ops.empty(nevex, 2 * g.nr)
        locked = self.ops.empty(nev, 2 * g.nc)
        sbasis = self.ops.empty(nev, 2 * g.nc)  # orthonormal basis of span(S Y_locked)
        nlock, lvals, lres, trace = 0, [], [], []
        converged, it_used, current, backups = False, 0, bounds, 0
        from .solver import MIXED_SWITCH, mixed_precision

        mixed, base_precision, filter_precisions = mixed_precision(), _lib.filter_precision(), []
        lam = res = act = None
        for it in range(1, cfg.maxiter + 1):
            it_used = it
            before = ledger.total_flops()
            k = nevex - nlock
            fcfg = FilterConfig.from_bounds(current, cfg.deg, cfg.plain_kernel_only)
            # precision policy of solver.py (complex64 filter, or the opt-in mixed policy)
            use_c64 = base_precision == "c64" or (
                mixed and (not trace or trace[-1].min_res_unlocked > MIXED_SWITCH * abs(bounds.mu_1)))
            filter_precisions.append("c64" if use_c64 else "c128")
            with ledger.timing("filter"):
                if second is not None:  # first iteration: the start block's second half arrives meanwhile
                    filt = self.chebyshev_c64 if use_c64 else (lambda x, f: self.chebyshev(x, f, row_buf))
                    filt(v[:k1], fcfg)
                    v[k1:] = start_block_finish(second.result(), k1, nevex, g, self.ops, self.c)
                    filt(v[k1:], fcfg)
                    second = None
                elif use_c64:
                    self.chebyshev_c64(v, fcfg)
                else:
                    self.chebyshev(v, fcfg, row_buf)
            ledger.add_flops("filter", cfg.deg * 8.0 * n * n * k)
            with ledger.timing("ortho"):
                v, _ = self.s_orthonormalize(v, sbasis[:nlock] if nlock else None)
            if nlock:
                ledger.add_flops("ortho", 16.0 * n * nlock * k)
            ledger.add_flops("ortho", 2 * (8.0 * n * k * k + 4.0 * n * k * k))
            from .solver import fused_residuals_for

            with ledger.timing("rr"):
                lam, vecs, lmm, fres, variant, fell_back = self.rayleigh_ritz(
                    v, row_buf, fused_residuals_for(cfg), cfg.rr_variant, it, ledger)
            backups += int(fell_back)
            with ledger.timing("residuals"):
                res = fres if fres is not None else self.residuals(vecs, lam, row_buf)
            ledger.add_flops("residuals", 8.0 * n * n * k)
            ritz = RitzSet(values=lam, vectors=None, residual_norms=res)
            new, act = lock_converged(ritz, tol, nev - nlock, normalizer)
            cnt = new.size
            if cnt:
                locked[nlock:nlock + cnt].copy_(vecs[:cnt])
                if nlock + cnt < nev:
                    with ledger.timing("ortho"):  # the reference's QR of S Y_locked is ortho time
                        self.extend_sbasis(sbasis, nlock, locked[nlock:nlock + cnt])
                nlock += cnt
                lvals.extend(lam[:cnt].tolist())
                lres.extend(res[:cnt].tolist())
            unl = res[act]
            trace.append(TraceRecord(it=it, locked=nlock, k=k, max_res=float(res.max()),
                                     min_res_unlocked=float(unl.min()) if unl.size else 0.0,
                                     mu_nevex=current.mu_nevex, variant=variant, lambda_min_m=lmm,
                                     flops=ledger.total_flops() - before))
            if nlock >= nev:
                converged = True
                break
            v = vecs[cnt:]
            act_vals = lam[act]
            still = act_vals[~ritz.converged[act]]
            cand = still if still.size else act_vals
            cand = np.minimum(cand[cand >= current.mu_1], 0.0)
            if cand.size:
                current = update_cutoff(current, cand)
        if converged:
            vals, blocks, resid = np.array(lvals), locked[:nlock], np.array(lres)
        else:
            miss = nev - nlock
            vals = np.concatenate([lvals, lam[act][:miss]])
            blocks = torch.cat([locked[:nlock], vecs[torch.as_tensor(act[:miss], device=vecs.device)]], dim=0)
            resid = np.concatenate([lres, res[act][:miss]])
        if pool is not None:
            pool.shutdown(wait=False)
        st.mark("iterations", nev)
        order = np.argsort(vals, kind="stable")[:nev]
        full = self.assemble_from_col(blocks[torch.as_tensor(order, device=blocks.device)].contiguous())
        st.mark("sort + assemble V", nev)
        out = SolveResult(lambdas=vals[order], v=full, residual_norms=resid[order], iterations_used=it_used,
                          converged=converged, trace=trace, bounds=bounds, ledger=ledger, backup_events=backups)
        out.filter_precisions = filter_precisions
        return out


def _start_share(grid: Grid, c_lo: int, c_hi: int, comm) -> tuple[list, int]:
    """Column edges of the p replicas' shares of columns [c_lo, c_hi) and the padded share width."""
    share = comm is not None and grid.p > 1
    edges = [c_lo + e for e in split(c_hi - c_lo, grid.p)] if share else [c_lo, c_hi]
    span = -(-(c_hi - c_lo) // grid.p) if share else c_hi - c_lo
    return edges, span


def start_block_host(seed: int, n: int, c_lo: int, c_hi: int, grid: Grid, comm=None) -> np.ndarray:
    """Host part of start_block_cols: this replica's share of columns [c_lo, c_hi), rows C_J of both
    halves, bit-exact (two contiguous counter ranges per column, rng.py:78-81), padded to the
    share width.  Pure numpy: safe to run on a helper thread while the GPU works."""
    edges, span = _start_share(grid, c_lo, c_hi, comm)
    me = grid.I if len(edges) > 2 else 0
    lo, hi = edges[me], edges[me + 1]
    m = grid.m
    col = np.arange(lo, hi, dtype=np.int64) * n
    part = np.zeros((span, 2 * grid.nc), dtype=np.complex128)
    if hi > lo and grid.nc:
        # the host's cores are shared by the ranks on this node (and each rank's driving thread)
        import os

        local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        nt = max(1, (os.cpu_count() or 1) // max(local, 1) - (1 if local > 1 else 0))
        part[:hi - lo, :grid.nc] = rng.complex_normals_segments(seed, col + grid.c0, grid.nc, threads=nt)
        part[:hi - lo, grid.nc:] = rng.complex_normals_segments(seed, col + m + grid.c0, grid.nc, threads=nt)
    return part


def start_block_finish(part: np.ndarray, c_lo: int, c_hi: int, grid: Grid, ops, comm=None):
    """Device part: upload this replica's share and allgather the shares over the column
    communicator (a collective: every rank calls it in the same order) -> (c_hi - c_lo, 2 nc)."""
    torch = ops.torch
    edges, span = _start_share(grid, c_lo, c_hi, comm)
    mine = torch.from_numpy(part).to(ops.device)
    if len(edges) == 2:
        return mine[:c_hi - c_lo].contiguous() if span != c_hi - c_lo else mine
    parts = comm.gather(mine, "col")
    return torch.cat([pt[:edges[i + 1] - edges[i]] for i, pt in enumerate(parts)], dim=0).contiguous()


def start_block_col(seed: int, n: int, cols: int, grid: Grid, ops, comm: "Comm | None" = None):
    """Rows C_J of both halves of the reference start block complex_normal_matrix(seed, n, cols)
    (solver.py:139-141), (cols, 2 nc) storage.  m <= EXACT_LIMIT: drawn bit-exactly on the host --
    the p replicas of a column group each draw a 1/p share of the columns and allgather them over the
    column communicator, so the grid draws the block exactly once (every rank drawing its full column
    slice made the N = 4 C3 solve pay 0.8 s of contended host time).  Above EXACT_LIMIT: the device
    rng (generate.py's policy)."""
    torch = ops.torch
    m = grid.m
    if m > EXACT_LIMIT and hasattr(ops, "ctx"):
        full = rng.device_complex_normal_matrix(seed, n, cols, ops.device).T  # (cols, n) storage rows
        return torch.cat([full[:, grid.c0:grid.c1], full[:, m + grid.c0:m + grid.c1]], dim=1).contiguous()
    return start_block_finish(start_block_host(seed, n, 0, cols, grid, comm), 0, cols, grid, ops, comm)


class DistributedSolver:
    """Holds the grid, the communicators and this rank's operator storage across solves (SPMD; every
    rank of an initialised torch.distributed world constructs it with the same Hamiltonian).
    ``source`` is a BseHamiltonian (host or device-born) or an (A, B) pair of host/device blocks, or
    a dict {"fwd": (A_t, B_t)} of this rank's own tile (A, B)[R_I, C_J].

    Storage (one decision for the whole grid: it depends only on settings every rank shares):
      * real-split (default, B != 0): the planes of the tile (A, B)[R_I, C_J] and nothing else,
        32 m^2 / (p q) bytes per GPU -- the paper's A/B-only layout; the transposed products read
        the same planes (bse_hop_tile_rs_t);
      * complex (B = 0, where the 3M kernel skips the B half, or planes=False): the complex tile and
        its block transpose (+ optional 3M sum planes)."""

    def __init__(self, source, *, m: int | None = None, device=None, grid: Grid | None = None, ops=None,
                 planes: bool | None = None):
        import torch

        world = torch.distributed.get_world_size() if torch.distributed.is_initialized() else 1
        rank = torch.distributed.get_rank() if torch.distributed.is_initialized() else 0
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.ops = ops or CudaOps(device)
        self.flags = 0
        if isinstance(source, dict):
            if m is None:
                raise ValidationError("m is required with pre-sliced tiles")
            self.flags = int(source.get("flags", 0))
        elif hasattr(source, "device_blocks"):
            m = source.m
            self.flags = source.flags
            if source.a is not None:
                source = (source.a, source.b)
            else:
                ab = source.device_blocks(device)
                source = (ab[:, :m], ab[:, m:])
        else:
            m = source[0].shape[0]
            b = source[1]
            self.flags = 0 if (bool(b.any()) if hasattr(b, "any") else True) else 1
        if planes is None:
            planes = _lib.uses_rs_planes() and not self.flags & 1
        self.use_planes = bool(planes) and hasattr(self.ops, "make_rs_planes")
        self.grid = grid or Grid(m, world, rank)
        self.comm = Comm(self.grid)
        self.load(source)

    @property
    def planes(self) -> bool:
        return self.inner.planes

    def load(self, source) -> None:
        """(Re)build this rank's operator storage (host -> device when the blocks are numpy)."""
        g = self.grid
        if isinstance(source, dict):
            fwd = tile_from_blocks(self.ops, *source["fwd"])
            trn = None if self.use_planes else tile_from_blocks(self.ops, *source["fwd"], transpose=True)
        else:
            fwd = slice_tile(self.ops, (g.r0, g.r1), (g.c0, g.c1), *source)
            trn = None if self.use_planes else slice_tile(self.ops, (g.c0, g.c1), (g.r0, g.r1), *source)
        if self.use_planes:
            self.fwd, self.trn = plane_tiles(self.ops, fwd)
            del fwd  # the complex tile was only the planes' source
        else:
            self.fwd, self.trn = fwd, trn
        self.inner = DistSolver(self.grid, self.comm, self.ops, self.fwd, self.trn)

    def operator_bytes(self) -> int:
        """Device bytes of this rank's operator storage."""
        if self.planes:
            return self.fwd.g.numel() * 8
        return sum(t.buf.numel() * ZB + (t.sd.numel() * ZB if t.sd is not None else 0) for t in (self.fwd, self.trn))

    def solve(self, cfg: SolverConfig) -> SolveResult:
        if hasattr(self.ops, "ctx"):
            self.ops.ctx.set_ham_flags(self.flags)
        g = self.inner.g
        if not self.planes and _lib.uses_sum_planes():
            # complex storage: optional 3M sum planes (bitwise-identical products without them)
            reserve = 6 * 16 * cfg.nevex * 2 * max(g.nr, g.nc)
            for t in (self.fwd, self.trn):
                if t.sd is None:
                    add_sum_planes(self.ops, t, reserve)
        res = self.inner.solve(cfg)
        res.v = res.v.T  # (n, nev) column-major view
        return res


def tile_blocks_host(grid: Grid, source) -> dict:
    """This rank's tile (A, B)[R_I, C_J] as host numpy arrays (F-order), from a BseHamiltonian or
    full (A, B) blocks -- the pre-sliced input a user hands DistributedSolver (bench e2e)."""
    if hasattr(source, "device_blocks"):
        if source.a is not None:
            a, b = source.a, source.b
        else:
            ab = source.device_blocks()
            a, b = ab[:, :source.m], ab[:, source.m:]
        flags = source.flags
    else:
        a, b = source
        flags = 0
    out = []
    for blk in (a, b):
        t = blk[grid.r0:grid.r1, grid.c0:grid.c1]
        t = t.T.contiguous().cpu().numpy().T if hasattr(t, "cpu") else np.asfortranarray(t)
        out.append(np.asfortranarray(t))
    return {"fwd": tuple(out), "flags": flags}


def solve_distributed(source, cfg: SolverConfig, *, device=None, grid: Grid | None = None, ops=None) -> SolveResult:
    """One-shot SPMD solve (see DistributedSolver); world size 1 runs the same code path."""
    return DistributedSolver(source, device=device, grid=grid, ops=ops).solve(cfg)
