"""Orthonormalisation of the filtered search space on the GPU.

Drop-in for bsesolve/ortho.py.  ``bse_s_orthonormalize`` projects the active
block against span(S Y_locked) (an orthonormal basis of it from CholQR2 on
the device instead of the reference's Householder QR — the projector is
basis independent), then runs CholeskyQR2 with the Gram products on the DMMA
GEMM; if the Gram Cholesky fails or max|Q*Q - I| > 1e-8 it falls back to
shifted CholeskyQR3 (replacing the Householder path, ortho.py:85-93,
113-128).  The column phase convention of ortho.py:70-82 is a per-column
reduction kernel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import RankDeficiencyError
from .hamiltonian import _device_for, _host_like, colmajor_empty, ld_of, to_colmajor
from .metrics import PhaseLedger

FALLBACK_TOL = 1e-8
RANK_TOL = 1e-10
_METHODS = {0: "cholqr", 1: "shifted_cholqr"}


@dataclass
class SearchSpace:
    """Locked columns followed by the active (orthonormal) block (ortho.py:31-67)."""

    q: object
    locked: int

    @property
    def n(self) -> int:
        return self.q.shape[0]

    @property
    def m(self) -> int:
        return self.q.shape[0] // 2

    @property
    def nevex(self) -> int:
        return self.q.shape[1]

    @property
    def active(self):
        return self.q[:, self.locked:]

    @property
    def locked_cols(self):
        return self.q[:, : self.locked]

    @property
    def q1(self):
        return self.q[: self.m]

    @property
    def q2(self):
        return self.q[self.m:]


def s_orthonormalize_inplace(v, locked_y=None, ledger: PhaseLedger | None = None) -> str:
    """In place on a column-major CUDA tensor v (n x k); locked_y (n x l) may be None."""
    n, k = v.shape
    l = 0 if locked_y is None else int(locked_y.shape[1])
    if k > n:
        raise RankDeficiencyError(f"cannot orthonormalize {k} columns in dimension {n}")
    method = ctypes.c_int(0)
    ctx = _lib.Context.get(v.device.index)
    yptr = _lib.dptr(locked_y) if l else ctypes.c_void_p(0)
    ctx.call("bse_s_orthonormalize", _lib.dptr(v), n, k, ld_of(v), yptr, l, ld_of(locked_y) if l else n,
             ctypes.byref(method))
    if ledger is not None:
        if l:
            ledger.add_flops("ortho", 16.0 * n * l * k)  # ortho.py:154
        ledger.add_flops("ortho", 2 * (8.0 * n * k * k + 4.0 * n * k * k))  # ortho.py:110
    return _METHODS[method.value]


def s_orthonormalize_basis_inplace(v, sbasis=None, ledger: PhaseLedger | None = None) -> str:
    """s_orthonormalize_inplace with the locked space given by its orthonormal basis (n x l,
    maintained by extend_sbasis): the solver loop's form (the reference's per-iteration QR of S Y
    is replaced by the incremental basis, same span)."""
    n, k = v.shape
    l = 0 if sbasis is None else int(sbasis.shape[1])
    if k > n:
        raise RankDeficiencyError(f"cannot orthonormalize {k} columns in dimension {n}")
    method = ctypes.c_int(0)
    ctx = _lib.Context.get(v.device.index)
    bptr = _lib.dptr(sbasis) if l else ctypes.c_void_p(0)
    ctx.call("bse_s_orthonormalize_basis", _lib.dptr(v), n, k, ld_of(v), bptr, l, ld_of(sbasis) if l else n,
             ctypes.byref(method))
    if ledger is not None:
        if l:
            ledger.add_flops("ortho", 16.0 * n * l * k)  # ortho.py:154 (the reference's model)
        ledger.add_flops("ortho", 2 * (8.0 * n * k * k + 4.0 * n * k * k))  # ortho.py:110
    return _METHODS[method.value]


def extend_sbasis(sbasis, l_old: int, y_new) -> None:
    """sbasis[:, l_old:l_old + c] <- orthonormal completion of span(S Y_new) against sbasis[:, :l_old]."""
    c = int(y_new.shape[1])
    if not c:
        return
    n = sbasis.shape[0]
    _lib.Context.get(sbasis.device.index).call("bse_extend_sbasis", _lib.dptr(sbasis), n, ld_of(sbasis), l_old,
                                               _lib.dptr(y_new), ld_of(y_new), c)


def fix_column_phases(q):
    """ortho.py:70-82 on the GPU (first entry >= 1e-8 max|q| made real positive)."""
    dev = _device_for(q)
    t = colmajor_empty(q.shape[0], q.shape[1], dev)
    t.copy_(to_colmajor(q, dev))
    _lib.Context.get(dev.index).call("bse_fix_phases", _lib.dptr(t), t.shape[0], t.shape[1], ld_of(t))
    return _host_like(q, t)


def cholqr_with_fallback(x, ledger: PhaseLedger | None = None):
    """Orthonormalize the columns of x; returns (Q, method) (ortho.py:96-129)."""
    dev = _device_for(x)
    t = colmajor_empty(x.shape[0], x.shape[1], dev)
    t.copy_(to_colmajor(x, dev))
    n, k = t.shape
    if k > n:
        raise RankDeficiencyError(f"cannot orthonormalize {k} columns in dimension {n}")
    if ledger is not None:
        ledger.add_flops("ortho", 2 * (8.0 * n * k * k + 4.0 * n * k * k))
    method = ctypes.c_int(0)
    _lib.Context.get(dev.index).call("bse_cholqr", _lib.dptr(t), n, k, ld_of(t), ctypes.byref(method))
    return _host_like(x, t), _METHODS[method.value]


def s_orthonormalize(vhat, locked_y=None, ledger: PhaseLedger | None = None):
    """ortho.py:132-158: returns (SearchSpace [Y_locked | Q_active], method)."""
    import torch

    dev = _device_for(vhat)
    v = colmajor_empty(vhat.shape[0], vhat.shape[1], dev)
    v.copy_(to_colmajor(vhat, dev))
    y = None
    if locked_y is not None and locked_y.shape[1]:
        y = to_colmajor(locked_y, dev)
    method = s_orthonormalize_inplace(v, y, ledger)
    q = v if y is None else torch.cat([y, v], dim=1)
    l = 0 if y is None else y.shape[1]
    return SearchSpace(q=_host_like(vhat, q), locked=l), method
