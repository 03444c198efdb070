"""Oblique Rayleigh-Ritz, residuals and locking on the GPU.

Drop-in for bsesolve/rayleigh_ritz.py.  ``bse_rr_hermitian`` forms
T = S H Q with the fused H-operator kernel (S flip in the epilogue),
W = Q^H T and M = I - 2 Q2^H Q2 on the DMMA GEMM, then solves the small
pencil on the device (Cholesky of W, two triangular solves, hermitian
eigensolver; cuSOLVER / cuBLAS on k x k) and back-transforms V = Q L^{-H} y
with column normalisation — the dual basis is never built
(rayleigh_ritz.py:98-143).  ``bse_residuals`` is the same H-operator GEMM
with a residual-norm epilogue (no H V block is ever written to HBM).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ValidationError
from .hamiltonian import BseHamiltonian, _device_for, _host_like, colmajor_empty, ld_of, to_colmajor
from .metrics import PhaseLedger

M_SINGULARITY_TOL = 1e-8
DIAG_ZERO_TOL = 1e-12


@dataclass
class ReducedProblem:
    """Reduced-problem record (rayleigh_ritz.py:41-51).  Inside the solver loop the k x k
    factors stay on the device (only the variant and |lambda|_min(Q*SQ) come back); the public
    build_hermitian_rq / build_backup_rq fill w, l, m, g (and d for the backup) as host arrays, as
    the reference returns them (rayleigh_ritz.py:140-143, 176-179)."""

    variant: str
    w: object = None
    l: object = None
    m: object = None
    g: object = None
    d: object = None
    lambda_min_m: float = float("nan")


@dataclass
class RitzSet:
    """Ascending Ritz values (host), unit Ritz vectors (device or host), residuals."""

    values: np.ndarray
    vectors: object
    residual_norms: np.ndarray | None = None
    converged: np.ndarray | None = None

    @property
    def k(self) -> int:
        return self.values.shape[0]


def _rr(entry: str, variant: str, ham: BseHamiltonian, q, ledger, fused_residuals: bool = False,
        capture: bool = False):
    n, k = q.shape
    lam = np.zeros(k)
    vout = colmajor_empty(n, k, q.device)
    lmm = ctypes.c_double(float("nan"))
    ab = ham.device_blocks(q.device)
    # the T = (S) H Q product runs on the real-split planes (csrc/hop_rs.cuh, registered for this call
    # only) when they are in use, else on the filter's 3M kernel when the sum planes are
    g = ham.device_rs_planes(q.device, reserve=3 * 16 * n * k) if _lib.uses_rs_planes() else None
    sdt = ham.device_sum_planes(q.device, reserve=2 * 16 * n * k) if _lib.uses_sum_planes() and g is None else None
    sd = _lib.dptr(sdt) if sdt is not None else None
    ctx = _lib.Context.get(q.device.index)
    res = np.zeros(k) if fused_residuals else None
    extra = (_lib.hptr(res) if fused_residuals else None,) if entry == "bse_rr_hermitian" else ()
    cap = None
    if capture:
        import torch

        cap = torch.zeros(4 * k * k + (k + 1) // 2, dtype=torch.complex128, device=q.device)
        ctx.call("bse_set_rr_capture", _lib.dptr(cap))
    try:
        if g is not None:  # ab is None when the operator is held as planes only
            ctx.call("bse_set_rs_planes", _lib.dptr(ab), ham.m, _lib.dptr(g), g.stride(1))
        ctx.call(entry, _lib.dptr(ab), sd, ld_of(ab) if ab is not None else ham.m, ham.m, _lib.dptr(q), ld_of(q), k,
                 _lib.hptr(lam), _lib.dptr(vout), ld_of(vout), ctypes.byref(lmm), *extra)
    finally:
        if g is not None:
            ctx.call("bse_set_rs_planes", None, 0, None, 0)
        if cap is not None:
            ctx.call("bse_set_rr_capture", None)
        if ledger is not None:
            # apply_h inside RR charges 8n^2k to "rr" (hamiltonian.py:148-150) before the model of
            # rayleigh_ritz.py:139 / :175 — the reference ledger counts both, so do we
            ledger.add_flops("rr", 8.0 * n * n * k)
    if ledger is not None:
        extra = (12.0 * n * k * k + 16.0 * k**3) if variant == "hermitian" else (20.0 * n * k * k + 30.0 * k**3)
        ledger.add_flops("rr", 8.0 * n * n * k + extra)
    red = ReducedProblem(variant=variant, lambda_min_m=lmm.value)
    if cap is not None:
        host = cap.cpu().numpy()
        kk = k * k
        w_, l_, m_, g_ = (host[i * kk:(i + 1) * kk].reshape(k, k, order="F") for i in range(4))
        red.w, red.m, red.g = w_.copy(), m_.copy(), g_.copy()
        if variant == "hermitian":
            red.l = np.tril(l_)
        else:
            red.d = host[4 * kk:].view(np.float64)[:k].copy()
    return RitzSet(values=lam, vectors=vout, residual_norms=res), red


def build_hermitian_rq_device(ham, q, ledger=None, fused_residuals: bool = False):
    """fused_residuals: also return ||H v - lam v|| computed as |S (S H Q) w / |Q w| - lam v|
    (saves the residual H application; differs from the explicit product at roundoff)."""
    return _rr("bse_rr_hermitian", "hermitian", ham, q, ledger, fused_residuals)


def build_backup_rq_device(ham, q, ledger=None):
    return _rr("bse_rr_backup", "backup", ham, q, ledger)


def _public(entry, variant, ham, q_active, ledger):
    dev = _device_for(q_active)
    q = to_colmajor(q_active, dev)
    ritz, red = _rr(entry, variant, ham, q, ledger, capture=True)
    ritz.vectors = _host_like(q_active, ritz.vectors)
    return ritz, red


def build_hermitian_rq(ham: BseHamiltonian, q_active, ledger: PhaseLedger | None = None):
    """Hermitian-equivalent projection (rayleigh_ritz.py:98-143)."""
    return _public("bse_rr_hermitian", "hermitian", ham, q_active, ledger)


def build_backup_rq(ham: BseHamiltonian, q_active, ledger: PhaseLedger | None = None):
    """Non-hermitian backup projection (rayleigh_ritz.py:146-179)."""
    return _public("bse_rr_backup", "backup", ham, q_active, ledger)


def residuals_device(ham: BseHamiltonian, values: np.ndarray, vectors, ledger=None) -> np.ndarray:
    n, k = vectors.shape
    out = np.zeros(k)
    lam = np.ascontiguousarray(values, dtype=np.float64)
    ab = ham.device_blocks(vectors.device)
    if ab is None:
        raise ValidationError("explicit residuals need the [A|B] blocks; a planes-only operator takes the fused "
                              "residuals of the RR (BSE200_RESIDUALS=fused)")
    _lib.Context.get(vectors.device.index).call(
        "bse_residuals", _lib.dptr(ab), ld_of(ab), ham.m, _lib.dptr(vectors), ld_of(vectors), k, _lib.hptr(lam),
        _lib.hptr(out))
    if ledger is not None:
        ledger.add_flops("residuals", 8.0 * n * n * k)
    return out


def residuals(ham: BseHamiltonian, ritz: RitzSet, ledger: PhaseLedger | None = None) -> np.ndarray:
    """||H v - lam v||_2 per column, stored on the RitzSet (rayleigh_ritz.py:182-190)."""
    dev = _device_for(ritz.vectors)
    v = to_colmajor(ritz.vectors, dev)
    ritz.residual_norms = residuals_device(ham, ritz.values, v, ledger)
    return ritz.residual_norms


def lock_converged(ritz: RitzSet, tol: float, nev: int, normalizer: float = 1.0):
    """Longest converged prefix, capped at nev (rayleigh_ritz.py:193-214); host scalars."""
    if ritz.residual_norms is None:
        raise ValidationError("residuals must be computed before locking")
    ok = ritz.residual_norms <= tol * normalizer
    ritz.converged = ok
    bad = np.flatnonzero(~ok[: min(nev, ritz.k)])
    count = int(bad[0]) if bad.size else min(nev, ritz.k)
    return np.arange(count), np.arange(count, ritz.k)
