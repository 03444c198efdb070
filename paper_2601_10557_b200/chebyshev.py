"""Scaled Chebyshev filter on the GPU (drop-in for bsesolve/chebyshev.py).

The whole degree-``deg`` filter is one C-ABI call (``bse_chebyshev_filter``):
``deg`` launches of the fused H-operator GEMM whose epilogue applies the
sigma-scaled three-term recurrence (chebyshev.py:58-74), rotating three
n x k device buffers.  No elementwise pass touches HBM between products.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .errors import ValidationError
from .hamiltonian import BseHamiltonian, _check_rows, _device_for, _host_like, colmajor_empty, ld_of, to_colmajor
from .lanczos import SpectralBounds
from .metrics import PhaseLedger


@dataclass(frozen=True)
class FilterConfig:
    """Center c, half width e, anchor s; even degree >= 2 (chebyshev.py:22-48)."""

    degree: int
    center: float
    half_width: float
    scale_ref: float
    plain_kernel_only: bool = False

    def __post_init__(self) -> None:
        if self.degree < 2 or self.degree % 2:
            raise ValidationError(f"filter degree must be even and >= 2, got {self.degree}")
        if not self.half_width > 0:
            raise ValidationError(f"filter half width must be positive, got {self.half_width}")

    @classmethod
    def from_bounds(cls, bounds: SpectralBounds, degree: int, plain_kernel_only: bool = False) -> "FilterConfig":
        return cls(degree=degree, center=(bounds.mu_n + bounds.mu_nevex) / 2.0,
                   half_width=(bounds.mu_n - bounds.mu_nevex) / 2.0, scale_ref=bounds.mu_1,
                   plain_kernel_only=plain_kernel_only)


def filter_inplace(ham: BseHamiltonian, v, cfg: FilterConfig, work=None, ledger: PhaseLedger | None = None):
    """p(H) v in place on a column-major complex128 CUDA tensor (n x k)."""
    n, k = v.shape
    if k == 0:
        return v
    if _lib.filter_precision() == "c64":
        return _filter_c64(ham, v, cfg, ledger)
    if work is None or work.numel() < 2 * ld_of(v) * k:
        import torch

        work = torch.empty(2 * ld_of(v) * k, dtype=torch.complex128, device=v.device)
    ab = ham.device_blocks(v.device)
    ctx = _lib.Context.get(v.device.index)
    if _lib.uses_rs_planes():
        # real-split filter: 4 n^2 k executed flops per step (csrc/hop_rs.cuh); the RR products run on
        # the same planes, so the 3M sum planes are only built when these are unavailable (B = 0, HBM)
        g = ham.device_rs_planes(v.device, reserve=2 * 16 * ld_of(v) * k)
        if g is not None:
            ctx.call("bse_chebyshev_filter_rs", _lib.dptr(g), g.stride(1), ham.m, _lib.dptr(v), ld_of(v), k,
                     cfg.degree, cfg.center, cfg.half_width, cfg.scale_ref, _lib.dptr(work))
            if ledger is not None:
                ledger.add_flops("filter", cfg.degree * 8.0 * n * n * k)
            return v
    # the planes must leave room for the RR's T and residual blocks (2 n k) next to the filter's buffers
    sdt = ham.device_sum_planes(v.device, reserve=2 * 16 * ld_of(v) * k) if _lib.uses_sum_planes() else None
    sd = _lib.dptr(sdt) if sdt is not None else None
    ctx.call("bse_chebyshev_filter", _lib.dptr(ab), sd, ld_of(ab), ham.m, _lib.dptr(v), ld_of(v), k, cfg.degree,
             cfg.center, cfg.half_width, cfg.scale_ref, _lib.dptr(work))
    if ledger is not None:
        ledger.add_flops("filter", cfg.degree * 8.0 * n * n * k)
    return v


def _filter_c64(ham: BseHamiltonian, v, cfg: FilterConfig, ledger):
    """complex64 filter on the tcgen05 tensor cores (3xTF32 products, FP32 recurrence)."""
    import torch

    n, k = v.shape
    m = ham.m
    mp = (m + 3) // 4 * 4
    pl = ham.device_c64_planes(v.device)
    work = torch.empty(48 * mp * k, dtype=torch.float32, device=v.device)
    ham.device_blocks(v.device)  # binds the Hamiltonian flags (B = 0)
    _lib.Context.get(v.device.index).call("bse_chebyshev_filter_c64", _lib.dptr(pl), m, _lib.dptr(v), ld_of(v), k,
                                          cfg.degree, cfg.center, cfg.half_width, cfg.scale_ref, _lib.dptr(work))
    if ledger is not None:
        ledger.add_flops("filter", cfg.degree * 8.0 * n * n * k)
    return v


def chebyshev_filter(ham: BseHamiltonian, vhat, cfg: FilterConfig, ledger: PhaseLedger | None = None):
    """Apply p(H) to the columns of vhat (chebyshev.py:51-75); returns a new array."""
    _check_rows(vhat, ham.n)
    dev = _device_for(vhat)
    v = to_colmajor(vhat, dev)
    out = colmajor_empty(v.shape[0], v.shape[1], dev)
    out.copy_(v)
    filter_inplace(ham, out, cfg, ledger=ledger)
    return _host_like(vhat, out)


def scalar_filter_value(lam: float, cfg: FilterConfig) -> float:
    """Gain of the filter at eigenvalue lam (chebyshev.py:78-89), host scalar."""
    c, e = cfg.center, cfg.half_width
    s1 = e / (cfg.scale_ref - c)
    s = s1
    prev, cur = 1.0, (lam - c) * (s1 / e)
    for _ in range(2, cfg.degree + 1):
        sn = 1.0 / (2.0 / s1 - s)
        prev, cur, s = cur, (2.0 * sn / e) * (lam - c) * cur - (s * sn) * prev, sn
    return cur
