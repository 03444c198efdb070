"""BSE Hamiltonian blocks on the device and the H / S / K / J operators.

Drop-in for bsesolve/hamiltonian.py.  ``BseHamiltonian`` keeps the reference
constructor contract (A hermitian, B symmetric, complex128, defects up to
1e-12 x scale repaired, larger ones rejected: hamiltonian.py:35-96) and adds
the device layout the kernels read: one m x 2m column-major complex128 buffer
``[A | B]`` per GPU (32 m^2 bytes, converted once; see DESIGN.md "HBM
layout").  ``apply_h`` and friends run on the GPU through the C ABI.
"""

from __future__ import annotations

import enum
import logging
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ValidationError
from .metrics import PhaseLedger

logger = logging.getLogger(__name__)

SYMMETRY_RTOL = 1e-12


class Definiteness(enum.Enum):
    UNKNOWN = "unknown"
    DEFINITE = "definite"
    INDEFINITE = "indefinite"


def as_complex_matrix(a, name: str = "matrix") -> np.ndarray:
    """2-D finite complex128, column-major (hamiltonian.py:35-42)."""
    arr = np.asfortranarray(a, dtype=np.complex128)
    if arr.ndim != 2:
        raise ValidationError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if arr.size and not np.isfinite(arr).all():
        raise ValidationError(f"{name} contains non-finite entries")
    return arr


def _repair(block: np.ndarray, mirror: np.ndarray, name: str, what: str) -> np.ndarray:
    """hamiltonian.py:45-60 semantics: exact -> as is; <= 1e-12 scale -> averaged; else reject."""
    if not block.size:
        return block
    gap = float(np.abs(block - mirror).max())
    if gap == 0.0:
        return block
    scale = float(np.abs(block).max())
    if scale > 0.0 and gap > SYMMETRY_RTOL * scale:
        raise ValidationError(
            f"{name} violates {what} beyond tolerance: defect={gap:.3e}, allowed={SYMMETRY_RTOL * scale:.3e}"
        )
    logger.warning("%s had a %s defect of %.3e (scale %.3e); symmetrized on load", name, what, gap, scale)
    return np.asfortranarray((block + mirror) / 2.0)


def _torch():
    import torch

    return torch


def colmajor_empty(rows: int, cols: int, device) -> "torch.Tensor":
    """Uninitialised column-major complex128 device matrix (shape rows x cols, strides (1, rows))."""
    torch = _torch()
    return torch.empty((cols, rows), dtype=torch.complex128, device=device).T


def to_colmajor(x, device) -> "torch.Tensor":
    """Column-major complex128 copy of a numpy / torch matrix on ``device``."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.complex128)
    else:
        arr = np.asarray(x, dtype=np.complex128)
        if arr.ndim == 1:
            arr = arr[:, None]
        t = torch.from_numpy(np.ascontiguousarray(arr.T)).to(device, non_blocking=False).T
        return t
    if t.ndim == 1:
        t = t[:, None]
    if t.stride(0) != 1 or t.stride(1) < t.shape[0]:
        t = t.T.contiguous().T
    return t


def ld_of(t) -> int:
    return max(int(t.stride(1)), int(t.shape[0]), 1) if t.ndim == 2 else int(t.shape[0])


@dataclass(eq=False)
class BseHamiltonian:
    """H = [[A, B], [-conj(B), -conj(A)]] stored as its blocks A and B.

    ``a``/``b`` are host numpy arrays (reference contract).  ``device_blocks``
    returns the ``[A | B]`` device buffer, uploaded once per device.  A
    Hamiltonian built on the GPU (``generate(..., device=...)``) may carry only
    the device copy; ``a``/``b`` are then downloaded lazily.
    """

    a: np.ndarray | None
    b: np.ndarray | None
    definiteness: Definiteness = field(default=Definiteness.UNKNOWN)

    def __post_init__(self) -> None:
        self._dev: dict = {}
        self._m = None
        if self.a is None and self.b is None:
            return  # device-born; populated by from_device()
        a = as_complex_matrix(self.a, "A")
        b = as_complex_matrix(self.b, "B")
        if a.shape[0] != a.shape[1] or b.shape[0] != b.shape[1]:
            raise ValidationError(f"blocks must be square, got {a.shape} and {b.shape}")
        if a.shape != b.shape:
            raise ValidationError(f"A and B must agree in size, got {a.shape} != {b.shape}")
        a = _repair(a, a.conj().T, "A", "hermiticity")
        b = _repair(b, b.T, "B", "symmetry")
        a.flags.writeable = False
        b.flags.writeable = False
        self.a, self.b = a, b
        self._m = a.shape[0]

    # ------------------------------------------------------------------ device
    @classmethod
    def from_device(cls, ab, definiteness: Definiteness = Definiteness.UNKNOWN) -> "BseHamiltonian":
        """Wrap an m x 2m column-major device buffer [A | B] (exactly hermitian / symmetric)."""
        ham = cls(None, None, definiteness)
        ham._m = int(ab.shape[0])
        ham._dev[ab.device] = ab
        return ham

    def device_blocks(self, device=None):
        """The [A | B] device buffer; None on a device where the operator is held as real-split
        planes only (planes_only / drop_blocks_for_planes)."""
        torch = _torch()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        device = torch.device(device)
        if device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        if device in self.__dict__.get("_planes_only", ()):
            _lib.Context.get(device.index).set_ham_flags(self.flags)
            return None
        ab = self._dev.get(device)
        if ab is None:
            if self.a is None:
                src = next(iter(self._dev.values()))
                ab = src.to(device)
                if ab.stride(0) != 1:
                    ab = ab.T.contiguous().T
            else:
                m = self.m
                ab = colmajor_empty(m, 2 * m, device)
                # F-ordered numpy -> (1, m)-strided host view -> one dense copy per block
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", UserWarning)  # read-only numpy views are only read here
                    ab[:, :m].copy_(torch.from_numpy(np.asfortranarray(self.a)))
                    ab[:, m:].copy_(torch.from_numpy(np.asfortranarray(self.b)))
            self._dev[device] = ab
        # every operator call fetches the blocks right before its C call: bind this Hamiltonian's flags
        _lib.Context.get(device.index).set_ham_flags(self.flags)
        return ab

    @property
    def b_is_zero(self) -> bool:
        """B == 0 exactly (TDA / hermitian limit): the operator then skips the B half."""
        z = self.__dict__.get("_bzero")
        if z is None:
            if self.b is not None:
                b = self.b  # cheap early exits before the full scan (typical B is dense)
                z = not (b.size and (b[0, 0] != 0 or b[-1, -1] != 0 or np.any(b[:, 0]) or np.any(b)))
            else:
                ab = next(iter(self._dev.values()))
                z = not bool((ab[:, self.m:] != 0).any().item())
            self._bzero = z
        return z

    @property
    def flags(self) -> int:
        return 1 if self.b_is_zero else 0  # BSE_HAM_B_ZERO

    def device_sum_planes(self, device, reserve: int = 0):
        """(re+im, re-im) planes of [A | B] for the 3M filter (bse_make_sum_planes), built once per device.
        None when they would not leave `reserve` bytes of HBM (e.g. n = 100k on one GPU: 80 GB of planes
        on top of 80 GB of blocks): the products then form the operand sums in registers (3M, same bits
        per output, ~7% slower)."""
        torch = _torch()
        device = torch.device(device)
        sd_cache = self.__dict__.setdefault("_sd", {})
        sd = sd_cache.get(device)
        if sd is False:
            return None
        if sd is None:
            ab = self.device_blocks(device)
            if not _lib.planes_fit(ab.numel() * 16, device, reserve):
                if device not in self.__dict__.setdefault("_sd_warned", set()):
                    self._sd_warned.add(device)
                    logger.warning("3M sum planes (%.1f GB) do not fit next to the solve; forming the operand sums "
                                   "in registers", ab.numel() * 16 / 1e9)
                return None  # decided again next call
            sd = colmajor_empty(ab.shape[0], ab.shape[1], device)
            _lib.Context.get(device.index).call("bse_make_sum_planes", _lib.dptr(ab), ld_of(ab), ab.shape[0],
                                                ab.shape[1], _lib.dptr(sd))
            sd_cache[device] = sd
        return sd

    def device_rs_planes(self, device, reserve: int = 0):
        """The four real planes [Ai + Bi | Ar - Br | Ar + Br | Ai - Bi] (m x 4m doubles, bse_make_rs_planes)
        of the real-split filter (csrc/hop_rs.cuh), built once per device; None when B == 0 (the 3M
        kernel skips the B half there) or when they would not leave `reserve` bytes of HBM."""
        torch = _torch()
        device = torch.device(device)
        cache = self.__dict__.setdefault("_rs", {})
        g = cache.get(device)
        if g is False:
            return None
        if g is None:
            ab = self.device_blocks(device)
            m = self.m
            ldg = m + (m & 1)
            if self.b_is_zero:
                cache[device] = False
                return None
            if not _lib.planes_fit(ldg * 4 * m * 8, device, reserve):
                return None  # decided again next call: HBM pressure is not a property of the operator
            g = torch.empty((4 * m, ldg), dtype=torch.float64, device=device).t()  # column-major m x 4m, ld ldg
            _lib.Context.get(device.index).call("bse_make_rs_planes", _lib.dptr(ab), ld_of(ab), m, m, _lib.dptr(g), ldg)
            cache[device] = g
        return g

    def device_c64_planes(self, device):
        """fp32 hi/lo planes of [A | B] in the K-major layout of the tcgen05 c64 filter
        (bse_c64_prepare; 32 m mp bytes), built once per device."""
        torch = _torch()
        device = torch.device(device)
        cache = self.__dict__.setdefault("_p64", {})
        pl = cache.get(device)
        if pl is None:
            ab = self.device_blocks(device)
            m = ab.shape[0]
            mp = (m + 3) // 4 * 4
            pl = torch.empty(4 * m * 2 * mp, dtype=torch.float32, device=device)
            _lib.Context.get(device.index).call("bse_c64_prepare", _lib.dptr(ab), ld_of(ab), m, _lib.dptr(pl))
            cache[device] = pl
        return pl

    def planes_only(self, device) -> bool:
        return _torch().device(device) in self.__dict__.get("_planes_only", ())

    def drop_blocks_for_planes(self, device) -> bool:
        """Hold the operator on `device` as its real-split planes only: build them (they carry the
        same 32 m^2 bytes of information) and free [A | B].  For n = 100k on one GPU, where [A | B]
        (80 GB) and the planes (80 GB) do not both fit beside the solve's vectors, so the
        real-split kernel runs every product (filter, RR, Lanczos) instead of 3M.  False when
        there is no room to build the planes even transiently, or B == 0."""
        torch = _torch()
        device = torch.device(device)
        if self.planes_only(device):
            return True
        if self.b_is_zero or not _lib.uses_rs_planes():
            return False
        self.flags  # noqa: B018 -- B == 0 is decided while the blocks still exist
        torch.cuda.empty_cache()
        if self.device_rs_planes(device) is None:
            return False
        self._dev.pop(device, None)
        self.__dict__.get("_sd", {}).pop(device, None)
        self.__dict__.get("_p64", {}).pop(device, None)
        self.__dict__.setdefault("_planes_only", set()).add(device)
        torch.cuda.empty_cache()
        return True

    def release_device(self) -> None:
        for cache in ("_sd", "_p64", "_rs"):
            self.__dict__.get(cache, {}).clear()
        if self.a is not None:
            self._dev.clear()
            self.__dict__.get("_planes_only", set()).clear()

    def host_blocks(self) -> tuple[np.ndarray, np.ndarray]:
        if self.a is None and not self._dev and self.__dict__.get("_planes_only"):
            # held as planes only: A, B back from Z, V, U, W (Ar = (V + U)/2, Br = (U - V)/2,
            # Ai = (Z + W)/2, Bi = (Z - W)/2) -- equal to the original blocks to rounding
            dev = next(iter(self._planes_only))
            g = self._rs[dev]
            m = self.m
            gm = g[:m]
            z, v, u, w = (gm[:, q * m:(q + 1) * m] for q in range(4))
            a = _torch().complex((v + u) * 0.5, (z + w) * 0.5)
            b = _torch().complex((u - v) * 0.5, (z - w) * 0.5)
            self.a = np.asfortranarray(a.T.contiguous().cpu().numpy().T)
            self.b = np.asfortranarray(b.T.contiguous().cpu().numpy().T)
            self.a.flags.writeable = False
            self.b.flags.writeable = False
        if self.a is None:
            ab = next(iter(self._dev.values()))
            m = self.m
            full = ab.T.contiguous().cpu().numpy().T  # F-order numpy
            self.a = np.asfortranarray(full[:, :m])
            self.b = np.asfortranarray(full[:, m:])
            self.a.flags.writeable = False
            self.b.flags.writeable = False
        return self.a, self.b

    @property
    def m(self) -> int:
        return self._m

    @property
    def n(self) -> int:
        return 2 * self._m


def _check_rows(x, n: int) -> None:
    if x.shape[0] != n:
        raise ValidationError(f"operand has {x.shape[0]} rows, expected {n}")


def _host_like(ref, t):
    """Return t as numpy when the caller passed numpy, else as a torch tensor."""
    torch = _torch()
    if isinstance(ref, torch.Tensor):
        return t
    return t.T.contiguous().cpu().numpy().T


def _device_for(x):
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------- S / K / J
def _halves(x, name: str):
    if x.shape[0] % 2:
        raise ValidationError(f"{name} needs an even row count, got {x.shape[0]}")
    return x.shape[0] // 2


def apply_s(x):
    """S x (hamiltonian.py:104-111): lower half negated."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        m = _halves(x, "S")
        out = x.clone()
        out[m:] *= -1.0
        return out
    x = np.asarray(x, dtype=np.complex128)
    m = _halves(x, "S")
    out = x.copy()
    out[m:] *= -1.0
    return out


def apply_k(x):
    """K x (hamiltonian.py:114-120): halves swapped."""
    torch = _torch()
    m = _halves(x, "K")
    if isinstance(x, torch.Tensor):
        return torch.cat([x[m:], x[:m]], dim=0)
    x = np.asarray(x, dtype=np.complex128)
    return np.concatenate([x[m:], x[:m]], axis=0)


def apply_j(x):
    """J x = (x_lower, -x_upper) (hamiltonian.py:123-129)."""
    torch = _torch()
    m = _halves(x, "J")
    if isinstance(x, torch.Tensor):
        return torch.cat([x[m:], -x[:m]], dim=0)
    x = np.asarray(x, dtype=np.complex128)
    return np.concatenate([x[m:], -x[:m]], axis=0)


# ---------------------------------------------------------------- H products
def _apply(ham: BseHamiltonian, x, low_sign: float, ledger, phase):
    vec = getattr(x, "ndim", 2) == 1
    _check_rows(x, ham.n)
    dev = _device_for(x)
    xd = to_colmajor(x, dev)
    k = xd.shape[1]
    y = colmajor_empty(ham.n, k, dev)
    ctx = _lib.Context.get(dev.index)
    ab = ham.device_blocks(dev)
    ctx.call("bse_apply_h", _lib.dptr(ab), None, ld_of(ab), ham.m, _lib.dptr(xd), ld_of(xd), _lib.dptr(y), ld_of(y),
             k, float(low_sign))
    if ledger is not None:
        ledger.add_flops(phase, 8.0 * ham.n * ham.n * k)
    out = _host_like(x, y)
    return out[:, 0] if vec else out


def apply_h(ham: BseHamiltonian, x, ledger: PhaseLedger | None = None, phase: str = "filter"):
    """H x on the GPU (hamiltonian.py:132-151): one fused DMMA GEMM over [A | B]."""
    return _apply(ham, x, 1.0, ledger, phase)


def apply_h_via_adjoint(ham: BseHamiltonian, x, ledger: PhaseLedger | None = None, phase: str = "filter"):
    """H x as S (H* (S x)) (hamiltonian.py:154-176).  On one device the
    adjoint identity is the same fused product (the block-transposed tiles
    only differ in the 2D-distributed layout)."""
    return _apply(ham, x, 1.0, ledger, phase)


def apply_sh(ham: BseHamiltonian, x, ledger: PhaseLedger | None = None, phase: str = "rr"):
    """S H x with the flip fused into the epilogue (rayleigh_ritz.py:112)."""
    return _apply(ham, x, -1.0, ledger, phase)


def materialize(ham: BseHamiltonian) -> np.ndarray:
    """Dense n x n H (oracles / structural checks only; hamiltonian.py:179-183)."""
    a, b = ham.host_blocks()
    return np.asfortranarray(np.block([[a, b], [-np.conj(b), -np.conj(a)]]))


def materialize_sh(ham: BseHamiltonian) -> np.ndarray:
    """Dense S H = [[A, B], [conj B, conj A]] (hamiltonian.py:186-190)."""
    a, b = ham.host_blocks()
    return np.asfortranarray(np.block([[a, b], [np.conj(b), np.conj(a)]]))


def validate_pseudo_hermitian(h_dense) -> tuple[bool, float]:
    """S H = H* S on a dense matrix (hamiltonian.py:193-205)."""
    h = np.asarray(h_dense, dtype=np.complex128)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValidationError(f"expected a square matrix, got shape {h.shape}")
    if h.shape[0] % 2:
        raise ValidationError(f"pseudo-hermitian structure needs even dimension, got {h.shape[0]}")
    lhs = apply_s(h)
    rhs = h.conj().T.copy()
    rhs[:, h.shape[0] // 2:] *= -1.0
    gap = float(np.abs(lhs - rhs).max()) if h.size else 0.0
    scale = float(np.abs(h).max()) if h.size else 0.0
    return gap <= SYMMETRY_RTOL * scale, gap


def is_definite(ham: BseHamiltonian) -> Definiteness:
    """Cholesky of S H on the device (hamiltonian.py:208-218), cached."""
    if ham.definiteness is not Definiteness.UNKNOWN:
        return ham.definiteness
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    ab = ham.device_blocks(dev)
    if ab is None:  # held as planes only: a temporary [A|B] (host copy, or rebuilt from the planes)
        a, b = ham.host_blocks()
        ab = colmajor_empty(ham.m, 2 * ham.m, dev)
        ab[:, :ham.m].copy_(torch.from_numpy(np.asfortranarray(a)))
        ab[:, ham.m:].copy_(torch.from_numpy(np.asfortranarray(b)))
    import ctypes

    flag = ctypes.c_int(0)
    _lib.Context.get(dev.index).call("bse_is_definite", _lib.dptr(ab), ld_of(ab), ham.m, ctypes.byref(flag))
    ham.definiteness = Definiteness.DEFINITE if flag.value else Definiteness.INDEFINITE
    return ham.definiteness
