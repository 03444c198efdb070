"""Spectral bounds from the sign-flip (S-inner-product) Lanczos recurrence.

Drop-in for bsesolve/lanczos.py.  The sweep (one H product per step plus two
S-dot products, lanczos.py:53-88) runs on the GPU through
``bse_lanczos_sweep``; the 24 x 24 tridiagonal eigenproblem and the density
cutoff (lanczos.py:127-164) are scalar host logic, as in the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np
import scipy.linalg as sla

from . import _lib, rng
from .errors import LanczosBreakdownError, ValidationError
from .hamiltonian import BseHamiltonian, ld_of
from .metrics import PhaseLedger

SAFETY_INFLATION = 0.01
MAX_RESTARTS = 3


@dataclass(frozen=True)
class SpectralBounds:
    """mu_1 <= mu_nevex <= mu_n with mu_n = -mu_1 (lanczos.py:36-50)."""

    mu_1: float
    mu_nevex: float
    mu_n: float
    steps: int
    ritz_values: np.ndarray
    ritz_weights: np.ndarray

    @property
    def nodes(self) -> list[tuple[float, float]]:
        return list(zip(self.ritz_values.tolist(), self.ritz_weights.tolist()))


def _sweep(ham: BseHamiltonian, start: np.ndarray, steps: int, ledger):
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    ab = ham.device_blocks(dev)
    alphas = np.zeros(steps)
    betas = np.zeros(max(steps - 1, 1))
    count = ctypes.c_int(0)
    st = np.ascontiguousarray(start, dtype=np.complex128)
    ctx = _lib.Context.get(dev.index)
    g = ham.device_rs_planes(dev) if ab is None else None  # planes-only operator: matvecs on the planes
    try:
        if g is not None:
            ctx.call("bse_set_rs_planes", None, ham.m, _lib.dptr(g), g.stride(1))
        ctx.call("bse_lanczos_sweep", _lib.dptr(ab), ld_of(ab) if ab is not None else ham.m, ham.m,
                 st.ctypes.data_as(ctypes.c_void_p), steps, _lib.hptr(alphas), _lib.hptr(betas), ctypes.byref(count))
    finally:
        if g is not None:
            ctx.call("bse_set_rs_planes", None, 0, None, 0)
    na = count.value
    # one H product for the start plus one per completed step (lanczos.py:58, 76)
    if ledger is not None:
        products = 1 + (na - 1 if na == steps else na)
        ledger.add_flops("lanczos", products * 8.0 * ham.n * ham.n)
    return alphas[:na], betas[: max(na - 1, 0)], na < steps


def _cutoff(theta: np.ndarray, weights: np.ndarray, nevex: int, n: int) -> float:
    """lanczos.py:145-164: midpoint past the node where the negative-axis weight reaches nevex/n."""
    neg = theta < 0
    if not neg.any():
        return 0.0
    cum = np.cumsum(weights[neg])
    hit = np.flatnonzero(cum >= nevex / n)
    j = int(hit[0]) if hit.size else int(neg.sum()) - 1
    return float((theta[j] + theta[j + 1]) / 2.0) if j + 1 < theta.shape[0] else float(theta[j])


def estimate_bounds(ham: BseHamiltonian, nevex: int, steps: int = 24, seed: int = 0,
                    ledger: PhaseLedger | None = None) -> SpectralBounds:
    """lanczos.py:91-142."""
    if steps < 2 or steps % 2:
        raise ValidationError(f"steps must be even and >= 2, got {steps}")
    if nevex < 0 or nevex > ham.n // 2:
        raise ValidationError(f"nevex must lie in [0, n/2], got {nevex}")
    al = be = np.empty(0)
    for attempt in range(MAX_RESTARTS + 1):
        start = rng.complex_normals(rng.substream(seed, attempt), ham.n)
        al, be, early = _sweep(ham, start, steps, ledger)
        if not early or len(al) >= min(4, steps):
            break
    if len(al) < min(4, steps):
        raise LanczosBreakdownError(
            f"Lanczos broke down before {min(4, steps)} steps on {MAX_RESTARTS + 1} start vectors")
    if len(al) % 2:
        al = al[:-1]
        be = be[: len(al) - 1]
    theta, y = sla.eigh_tridiagonal(al, be)
    weights = y[0, :] ** 2
    mu_1 = float(theta[0]) - SAFETY_INFLATION * abs(float(theta[0]))
    mu_n = -mu_1
    cut = float(min(max(_cutoff(theta, weights, nevex, ham.n), mu_1), mu_n))
    return SpectralBounds(mu_1=mu_1, mu_nevex=cut, mu_n=mu_n, steps=len(al), ritz_values=theta,
                          ritz_weights=weights)


def update_cutoff(bounds: SpectralBounds, nonconverged_ritz) -> SpectralBounds:
    """lanczos.py:167-181: new mu_nevex = max non-converged Ritz value (ignored if >= mu_n)."""
    values = np.asarray(nonconverged_ritz, dtype=np.float64)
    if values.size == 0:
        raise ValidationError("update_cutoff needs at least one Ritz value")
    top = float(values.max())
    if not top < bounds.mu_n:
        return bounds
    return replace(bounds, mu_nevex=max(top, bounds.mu_1))
