"""Synthetic definite BSE Hamiltonians built on the GPU.

Same construction as bsesolve/generate.py:60-83 —
A = C C^H + alpha I (hermitised), B = ratio * lambda_min(A) / ||B0||_2 * B0 with
B0 = (D + D^T)/2, C and D complex-normal streams of tags 0 and 1 — but every
O(m^3) step runs on the device: C C^H on the DMMA GEMM, the eigen/singular
value scalars with cuSOLVER, the stream draws with the bit-exact splitmix64
kernel.  Where the CPU reference needs ~1 h and 75 GB at m = 20,000 this takes
seconds, and m = 50,000 (n = 100k, configs C4) fits one B200.

Exactness policy:
  * m <= EXACT_LIMIT (32,768; covers C1, C2 and the headline C3): the
    reference's instance.  C and D are drawn on the host with the reference
    stream (bit-identical normals), lambda_min(A) and ||B0||_2 come from dense
    device eigensolvers (values-only heevd of A and of B0^H B0; they differ
    from LAPACK's eigvalsh/svdvals at roundoff, tests/test_gpu_large_parity.py
    checks them against the reference's own scalars at C2/C3), and the
    definiteness of S H is verified by the device Cholesky of the n x n S H,
    as generate.py:77 does.  A = C C^H differs from numpy's only by the
    GEMM summation order (<= 1e-15 relative).
  * m > EXACT_LIMIT (C4, n = 100k, where the dense eigensolvers do not fit
    beside [A|B]): normals drawn on the device (words bit-exact, Box-Muller
    within ~1 ulp), lambda_min(A) replaced by its certified lower bound
    alpha, ||B0||_2 by a 200-step power-iteration estimate; S H is positive
    definite by construction (||B||_2 <= ratio * alpha < lambda_min(A)), so
    no n x n Cholesky is run.  The reference cannot build this size in
    reasonable time either.
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
EXACT_LIMIT = 32768


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
        pool = draw_d = None
        if exact:
            from concurrent.futures import ThreadPoolExecutor

            # the host draws D (tag 1) while the device works on A
            pool = ThreadPoolExecutor(1)
            if spec.coupling_ratio != 0.0:
                draw_d = pool.submit(rng.complex_normals, rng.substream(spec.seed, TAG_COUPLING), m * m)
            z = torch.from_numpy(rng.complex_normals(seed_c, m * m)).to(device)  # C, column-major
            tmp.view(m, m).copy_(z.view(m, m).T)  # row-major C = column-major C^T
            del z
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
            if exact:
                tmp.copy_(torch.from_numpy(draw_d.result()))  # D, column-major
            else:
                ctx.call("bse_complex_normals", _lib.dptr(tmp), ctypes.c_uint64(rng.substream(spec.seed, TAG_COUPLING)),
                         0, m * m)
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
        # release the m^2 scratch now: a cached segment later partly reused by small tensors can no
        # longer be returned, which is what kept n = 100k from building its planes on one GPU
        torch.cuda.empty_cache()
        if pool is not None:
            pool.shutdown()
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
