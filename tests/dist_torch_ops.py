"""Torch (CPU) reference implementation of the device ops of
paper_2601_10557_b200/dist.py, so the 2D-distributed algorithm (layouts,
diagonal shift folding, reductions, gathers) can be checked under gloo with
world_size 2 / 4 on a machine without GPUs.  TEST INFRASTRUCTURE."""
import numpy as np
import torch


class TorchOps:
    def __init__(self):
        self.torch = torch
        self.device = torch.device("cpu")

    def empty(self, k, rows):
        return torch.empty((k, rows), dtype=torch.complex128)

    @staticmethod
    def _mat(tile):
        kc = tile.kc
        return tile.buf[:kc].T, tile.buf[kc:2 * kc].T  # (mr x kc) A_t, B_t

    # real-split storage (csrc/hop_rs.cuh): planes Z, V, U, W of a tile, one (4 kc, ldg) float64 storage
    def make_rs_planes(self, tile):
        at, bt = self._mat(tile)
        mr, kc = tile.mr, tile.kc
        ldg = mr + (mr & 1)
        g = torch.zeros((4 * kc, ldg), dtype=torch.float64)
        gm = g.t()
        for q, pl in enumerate((at.imag + bt.imag, at.real - bt.real, at.real + bt.real, at.imag - bt.imag)):
            gm[:mr, q * kc:(q + 1) * kc] = pl
        return g, ldg

    @staticmethod
    def _rs_product(tile, xf, yf):
        """folded product: forward x' = i Z x + V y, y' = U x + i W y; transposed (same planes)
        x' = -i W^T x + V^T y, y' = U^T x - i Z^T y."""
        gm = tile.g.t()
        if tile.trans:
            rows, cols = tile.kc, tile.mr  # the planes' own shape
            z, v, u, w = (gm[:rows, q * cols:(q + 1) * cols].to(torch.complex128) for q in range(4))
            return -1j * (w.T @ xf) + v.T @ yf, u.T @ xf - 1j * (z.T @ yf)
        z, v, u, w = (gm[:tile.mr, q * tile.kc:(q + 1) * tile.kc].to(torch.complex128) for q in range(4))
        return 1j * (z @ xf) + v @ yf, u @ xf + 1j * (w @ yf)

    def rs_fold(self, v, rows, scale, scale2=None, out=None):
        out = v if out is None else out
        s2 = scale if scale2 is None else scale2
        x1, x2 = v[:, :rows].clone(), v[:, rows:2 * rows].clone()
        out[:, :rows] = scale * (x1 + x2)
        out[:, rows:2 * rows] = s2 * (x1 - x2)

    def hop(self, tile, x, y, *, alpha=1.0, shift=0.0, shift_col=None, shift_rows=(0, 0), s_off=0, beta=0.0,
            p=None, low_sign=1.0, filter=False, rs=False):
        mr, kc = tile.mr, tile.kc
        x1, x2 = x[:, :kc].T, x[:, kc:2 * kc].T
        if rs:
            assert low_sign == 1.0
            up, low = self._rs_product(tile, x1, x2)
        else:
            at, bt = self._mat(tile)
            up = at @ x1 + bt @ x2
            low = -(at.conj() @ x2 + bt.conj() @ x1)
        lo, hi = shift_rows
        if (shift != 0.0 or shift_col is not None) and hi > lo:
            sh = shift_col[None, :] if shift_col is not None else shift
            up[lo:hi] = up[lo:hi] - sh * x1[lo + s_off:hi + s_off]
            low[lo:hi] = low[lo:hi] - sh * x2[lo + s_off:hi + s_off]
        up, low = alpha * up, alpha * low
        if beta != 0.0:
            up = up - beta * p[:, :mr].T
            low = low - beta * p[:, mr:2 * mr].T
        low = low * low_sign
        y[:, :mr] = up.T
        y[:, mr:2 * mr] = low.T

    # complex64 filter emulation (dist.DistSolver.chebyshev_c64): a "plane set" is a complex64
    # (k, 2 rows) block, the product is formed in complex128 and rounded to complex64 like the
    # fp32 tile product; the raw buffer is a flat complex64 array (contiguous views for gloo)
    def c64_planes(self, rows, k):
        return torch.empty((k, 2 * rows), dtype=torch.complex64)

    def c64_raw(self, rows, k):
        return torch.empty(k * 2 * rows, dtype=torch.complex64)

    def c64_raw_view(self, raw, rows, k):
        return raw[:k * 2 * rows].view(k, 2 * rows)

    def c64_tile_planes(self, tile, src):
        return tile

    def c64_to_planes(self, v, rows, planes):
        planes.copy_(v.to(torch.complex64))

    def c64_from_planes(self, planes, rows, v):
        v.copy_(planes.to(torch.complex128))

    def c64_step(self, pplanes, tile, k, x, out, *, alpha, shift, shift_rows, s_off, beta=0.0, prev=None):
        y = torch.empty((k, 2 * tile.mr), dtype=torch.complex128)
        self.hop(pplanes, x.to(torch.complex128), y, alpha=alpha, shift=shift, shift_rows=shift_rows, s_off=s_off,
                 beta=beta, p=prev.to(torch.complex128) if prev is not None else None)
        self.c64_raw_view(out, tile.mr, k).copy_(y.to(torch.complex64))

    def c64_split(self, raw, rows, k, planes):
        planes.copy_(self.c64_raw_view(raw, rows, k))

    def gram(self, a, b):
        return (a.conj() @ b.T).T.contiguous()  # storage (k2, k1) of a^H b

    def nn(self, a, w, out=None, alpha=1.0, beta=0.0):
        r = alpha * (a.T @ w.T)
        if out is None:
            return r.T.contiguous()
        out.copy_((r + beta * out.T).T)
        return out

    def chol_rinv(self, g, shift=0.0, rdiag=None):
        gm = g.T
        gm = (gm + gm.conj().T) / 2 + shift * torch.eye(gm.shape[0], dtype=gm.dtype)
        r, info = torch.linalg.cholesky_ex(gm, upper=True)
        if int(info) != 0:
            return None, int(info)
        if rdiag is not None:
            rdiag.copy_(torch.diagonal(r).abs())
        return torch.linalg.inv(r).T.contiguous(), 0

    def rr_backup_pencil(self, g0, w, g2):
        """rayleigh_ritz.py:160-175 on the summed k x k partials (storage = transposes)."""
        k = w.shape[0]
        mm = torch.eye(k, dtype=w.dtype) - 2 * g2.T
        mm = (mm + mm.conj().T) / 2
        lmm = float(torch.linalg.eigvalsh(mm).abs().min())
        d = torch.real(torch.diagonal(mm)).clone()
        d[d.abs() <= 1e-12] = 1.0
        off = mm - torch.diag(torch.diagonal(mm))
        g = (g0.T - off @ w.T) / d[:, None]
        vals, y = np.linalg.eig(g.numpy())
        order = np.argsort(vals.real, kind="stable")
        return vals.real[order].copy(), torch.from_numpy(y[:, order]).T.contiguous(), lmm

    def rr_pencil_part(self, part, w, g2):
        """The two halves of rr_pencil (bse_rr_pencil_part)."""
        if part == 1:
            k = w.shape[0]
            mm = torch.eye(k, dtype=w.dtype) - 2 * g2.T
            return float(torch.linalg.eigvalsh((mm + mm.conj().T) / 2).abs().min())
        lam, wv, _ = self.rr_pencil(w, g2, check_m=False)
        return lam, wv

    def rr_pencil(self, w, g2, check_m=True):
        from paper_2601_10557_b200.errors import HermitianRqError

        wm = w.T
        wm = (wm + wm.conj().T) / 2
        k = wm.shape[0]
        mm = torch.eye(k, dtype=wm.dtype) - 2 * g2.T
        mm = (mm + mm.conj().T) / 2
        lmm = float(torch.linalg.eigvalsh(mm).abs().min()) if check_m else float("nan")
        if check_m and lmm < 1e-8:
            raise HermitianRqError("M singular")
        ell, info = torch.linalg.cholesky_ex(wm)
        if int(info):
            raise HermitianRqError("Cholesky of Q*SHQ failed (W not definite)")
        gg = torch.linalg.solve_triangular(ell, mm, upper=False)
        gg = torch.linalg.solve_triangular(ell, gg.conj().T, upper=False).conj().T
        gg = (gg + gg.conj().T) / 2
        th, y = torch.linalg.eigh(gg)
        lam = 1.0 / th.numpy()
        order = np.argsort(lam, kind="stable")
        wv = torch.linalg.solve_triangular(ell.conj().T, y, upper=True)[:, torch.as_tensor(order)]
        return lam[order], wv.T.contiguous(), lmm

    def resid_partial(self, u, v, half, uscale, lam):
        sg = torch.ones(u.shape[1], dtype=torch.float64)
        sg[half:] = -1.0
        r = sg[None, :] * u * uscale[:, None] - lam[:, None] * v
        return (r.real ** 2 + r.imag ** 2).sum(dim=1)

    def colnorm2(self, x):
        return (x.real ** 2 + x.imag ** 2).sum(dim=1)

    def colscale_rsqrt(self, x, n2):
        x /= torch.sqrt(n2)[:, None]

    def defect(self, g):
        return float((g.T - torch.eye(g.shape[0], dtype=g.dtype)).abs().max())

    def sflip(self, x):
        y = x.clone()
        y[:, x.shape[1] // 2:] *= -1
        return y
