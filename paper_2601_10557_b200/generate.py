"""Synthetic definite BSE Hamiltonians built on the GPU.

Same construction as bsesolve/generate.py:60-83 —
A = C C^H + alpha I (hermitised), B = ratio * lambda_min(A) / ||B0||_2 * B0 with
B0 = (D + D^T)/2, C and D complex-normal streams of tags 0 and 1 — but every
O(m^3) step runs on the device: C C^H on the DMMA GEMM, the eigen/singular
value scalars with cuSOLVER, the stream draws with the bit-exact splitmix64
kernel.  Where the CPU reference needs ~1 h and 75 GB at m = 20,000 this takes
seconds, and m = 50,000 (n = 100k, configs C4) fits one B200.

Exactness policy:
  * m <= EXACT_LIMIT: normals drawn on the host (bit-identical to the
    reference), lambda_min(A) and ||B0||_2 from dense device eigensolvers
    (differences vs. LAPACK at roundoff), definiteness verified by the
    device Cholesky of S H as the reference does (generate.py:77).
  * m > EXACT_LIMIT: normals drawn on the device (words bit-exact,
    Box-Muller within ~1 ulp), lambda_min(A) replaced by its certified lower
    bound alpha, ||B0||_2 by a 200-step power-iteration estimate; S H is
    positive definite by construction (||B||_2 <= ratio * alpha < lambda_min(A)
    for ratio < 1 as long as the estimate is within 1/ratio of the true
    norm), so no n x n Cholesky is run.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, rng
from .errors import ValidationError
from .hamiltonian import BseHamiltonian, Definiteness, colmajor_empty, is_definite

TAG_RESONANT = 0
TAG_COUPLING = 1
EXACT_LIMIT = 4096


@dataclass(frozen=True)
class GeneratorSpec:
    """generate.py:35-57."""

    m: int
    seed: int
    alpha: float = 1.0
    coupling_ratio: float = 0.5
    mode: str = "definite"

    def __post_init__(self) -> None:
        if self.m < 1:
            raise ValidationError(f"m must be >= 1, got {self.m}")
        if self.alpha <= 0:
            raise ValidationError(f"alpha must be positive, got {self.alpha}")
        if self.coupling_ratio < 0:
            raise ValidationError(f"coupling_ratio must be >= 0, got {self.coupling_ratio}")
        if self.mode not in ("definite", "indefinite"):
            raise ValidationError(f"mode must be definite or indefinite, got {self.mode!r}")
        if self.mode == "definite" and self.coupling_ratio >= 1:
            raise ValidationError(f"definite mode requires coupling_ratio < 1, got {self.coupling_ratio}")


def _normals_into(ctx, buf_flat, seed: int, count: int, host: bool) -> None:
    import torch

    if host:
        z = rng.complex_normals(seed, count)
        buf_flat.copy_(torch.from_numpy(z))
    else:
        ctx.call("bse_complex_normals", _lib.dptr(buf_flat), ctypes.c_uint64(seed), 0, count)


def _power_norm(ctx, b0, m: int, iters: int = 200) -> float:
    """||B0||_2 estimate: power iteration on B0^H B0 (device GEMMs, k = 1)."""
    import torch

    x = torch.from_numpy(rng.complex_normals(rng.substream(12345, 7), m)).to(b0.device)[:, None]
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    est = 0.0
    for _ in range(iters):
        x = x / torch.linalg.vector_norm(x)
        ctx.call("bse_zgemm_nn", m, 1, m, 1.0, _lib.dptr(b0), m, _lib.dptr(x), m, 0.0, _lib.dptr(y), m)
        ctx.call("bse_zgemm_cn", m, 1, m, 1.0, _lib.dptr(b0), m, _lib.dptr(y), m, 0.0, _lib.dptr(z), m)
        est = float(torch.sqrt(torch.linalg.vector_norm(z)).item())
        x, z = z, x
    return est


def generate(spec: GeneratorSpec, device=None, exact: bool | None = None) -> BseHamiltonian:
    """Build the Hamiltonian described by spec on the GPU (deterministic per seed)."""
    import torch

    m = spec.m
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    exact = m <= EXACT_LIMIT if exact is None else exact
    ctx = _lib.Context.get(device.index)
    with torch.cuda.device(device):
        ab = colmajor_empty(m, 2 * m, device)
        a = ab[:, :m]
        b = ab[:, m:]
        tmp = torch.empty(m * m, dtype=torch.complex128, device=device)
        # tmp <- Ct = C^T column-major (Ct[l, i] = C[i, l]) so that conj(C C^H) = Ct^H Ct
        seed_c = rng.substream(spec.seed, TAG_RESONANT)
        if exact:
            ct = np.asfortranarray(rng.complex_normal_matrix(seed_c, m, m).T)
            tmp.copy_(torch.from_numpy(ct.reshape(-1, order="F")))
        else:
            ctx.call("bse_complex_normals_t", _lib.dptr(tmp), ctypes.c_uint64(seed_c), m, m)
        # conj(A) = Ct^H Ct  ->  A = conj(.) + alpha I, hermitised (generate.py:64-65)
        ctx.call("bse_zgemm_cn", m, m, m, 1.0, _lib.dptr(tmp), m, _lib.dptr(tmp), m, 0.0, _lib.dptr(a), m)
        ctx.call("bse_scale_shift", _lib.dptr(a), m, m, 1.0, float(spec.alpha), 1)
        ctx.call("bse_symmetrize", _lib.dptr(a), m, m, 1)
        info = {"exact": exact}
        if spec.coupling_ratio == 0.0:
            b.zero_()
        else:
            _normals_into(ctx, tmp, rng.substream(spec.seed, TAG_COUPLING), m * m, exact)
            ctx.call("bse_symmetrize", _lib.dptr(tmp), m, m, 0)  # B0 = (D + D^T)/2, column-major in tmp
            if exact:
                w = np.zeros(m)
                ctx.call("bse_eigvalsh", _lib.dptr(a), m, m, _lib.hptr(w))
                lam_min = float(w[0])
                gram = torch.empty(m * m, dtype=torch.complex128, device=device)
                ctx.call("bse_zgemm_cn", m, m, m, 1.0, _lib.dptr(tmp), m, _lib.dptr(tmp), m, 0.0, _lib.dptr(gram), m)
                ctx.call("bse_eigvalsh", _lib.dptr(gram), m, m, _lib.hptr(w))
                del gram
                b_norm = float(np.sqrt(max(w[-1], 0.0)))
            else:
                lam_min = float(spec.alpha)
                b_norm = _power_norm(ctx, tmp, m)
            info.update(lambda_min_a=lam_min, b0_norm=b_norm)
            scale = spec.coupling_ratio * lam_min / b_norm
            b.copy_(tmp.view(m, m).T)  # column-major B0
            ctx.call("bse_scale_shift", _lib.dptr(b), m, m, float(scale), 0.0, 0)
        del tmp
        definite = Definiteness.UNKNOWN
        if spec.mode == "definite" and not exact:
            definite = Definiteness.DEFINITE  # certified by construction (module docstring)
        ham = BseHamiltonian.from_device(ab, definite)
        ham.construction = info
        if exact:
            outcome = is_definite(ham)
            if spec.mode == "definite" and outcome is not Definiteness.DEFINITE:
                raise AssertionError(
                    f"internal error: certified definite construction failed the Cholesky check (m={m}, seed={spec.seed})")
    return ham
