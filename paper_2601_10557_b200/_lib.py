"""ctypes binding of the bse200 C ABI (include/bse200.h).

This is the only door to the GPU: every numerical step of the solve goes
through ``libbse200.so``.  There is no CPU fallback — if the library or a CUDA
device is missing, every entry point raises ``RuntimeError`` loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (
    HermitianRqError,
    IndefiniteError,
    LanczosBreakdownError,
    NumericalError,
    RankDeficiencyError,
    ValidationError,
)

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("BSE200_LIB", _HERE / "libbse200.so"))

_i64 = C.c_int64
_vp = C.c_void_p
_dbl = C.c_double
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

class HopTileArgs(C.Structure):
    """bse_hop_tile_args (include/bse200.h)."""

    _fields_ = [
        ("pa", _vp), ("pb", _vp), ("sa", _vp), ("sb", _vp), ("lda", _i64), ("mr", _i64), ("kc", _i64),
        ("x1", _vp), ("x2", _vp), ("ldx", _i64), ("k", _i64),
        ("y1", _vp), ("y2", _vp), ("ldy", _i64),
        ("s1", _vp), ("s2", _vp), ("lds", _i64), ("shift_lo", _i64), ("shift_hi", _i64),
        ("shift", _dbl), ("d_shift_col", _vp),
        ("p1", _vp), ("p2", _vp), ("ldp", _i64),
        ("alpha", _dbl), ("beta", _dbl), ("low_sign", _dbl), ("filter", C.c_int),
    ]


class C64TileArgs(C.Structure):
    """bse_c64_tile_args (include/bse200.h)."""

    _fields_ = [
        ("pplanes", _vp), ("mo", _i64), ("kc", _i64), ("k", _i64),
        ("x", _vp), ("prev", _vp), ("out", _vp),
        ("alpha", _dbl), ("beta", _dbl), ("shift", _dbl),
        ("shift_lo", _i64), ("shift_hi", _i64), ("s_off", _i64), ("raw", C.c_int),
    ]


# name -> (restype, argtypes); mirrors include/bse200.h
_SIGS = {
    "bse_version": (C.c_char_p, []),
    "bse_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "bse_ctx_destroy": (None, [_vp]),
    "bse_set_stream": (C.c_int, [_vp, _vp]),
    "bse_set_filter_algorithm": (C.c_int, [_vp, C.c_int]),
    "bse_set_hamiltonian_flags": (C.c_int, [_vp, C.c_uint]),
    "bse_last_error": (C.c_char_p, [_vp]),
    "bse_launch_count": (_i64, [_vp]),
    "bse_apply_h": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _dbl]),
    "bse_filter_step": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _i64, _dbl, _dbl, _dbl]),
    "bse_chebyshev_filter": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, C.c_int, _dbl, _dbl, _dbl, _vp]),
    "bse_make_sum_planes": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "bse_make_rs_planes": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64]),
    "bse_set_rs_planes": (C.c_int, [_vp, _vp, _i64, _vp, _i64]),
    "bse_chebyshev_filter_rs": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, C.c_int, _dbl, _dbl, _dbl, _vp]),
    "bse_residuals": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _dp, _dp]),
    "bse_s_orthonormalize": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _ip]),
    "bse_cholqr": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _ip]),
    "bse_fix_phases": (C.c_int, [_vp, _vp, _i64, _i64, _i64]),
    "bse_rr_hermitian": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _dp, _vp, _i64, _dp, _dp]),
    "bse_rr_backup": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _dp, _vp, _i64, _dp]),
    "bse_lanczos_sweep": (C.c_int, [_vp, _vp, _i64, _i64, _vp, C.c_int, _dp, _dp, _ip]),
    "bse_is_definite": (C.c_int, [_vp, _vp, _i64, _i64, _ip]),
    "bse_hop_tile": (C.c_int, [_vp, C.POINTER(HopTileArgs)]),
    "bse_hop_tile_rs": (C.c_int, [_vp, C.POINTER(HopTileArgs), _vp, _i64]),
    "bse_hop_tile_rs_t": (C.c_int, [_vp, C.POINTER(HopTileArgs), _vp, _i64]),
    "bse_set_push_targets": (C.c_int, [_vp, C.POINTER(_vp), C.c_int]),
    "bse_group_sum": (C.c_int, [_vp, _vp, _i64, C.c_int, _vp, _i64]),
    "bse_set_rr_capture": (C.c_int, [_vp, _vp]),
    "bse_extend_sbasis": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64]),
    "bse_s_orthonormalize_basis": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _ip]),
    "bse_rs_fold": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _dbl, _dbl]),
    "bse_c64_tile_planes": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "bse_c64_tile_step": (C.c_int, [_vp, C.POINTER(C64TileArgs)]),
    "bse_c64_split": (C.c_int, [_vp, _vp, _i64, _i64, _vp]),
    "bse_c64_to_planes": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "bse_c64_from_planes": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64]),
    "bse_chol_rinv": (C.c_int, [_vp, _vp, _i64, _dbl, _vp, _vp, _ip]),
    "bse_rr_pencil": (C.c_int, [_vp, _vp, _vp, _i64, _dp, _vp, _dp]),
    "bse_rr_pencil_part": (C.c_int, [_vp, C.c_int, _vp, _vp, _i64, _dp, _vp, _dp]),
    "bse_rr_backup_pencil": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _dp, _vp, _dp]),
    "bse_resid_partial": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "bse_colnorm2": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "bse_colscale_rsqrt": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "bse_defect": (C.c_int, [_vp, _vp, _i64, _dp]),
    "bse_sflip": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _i64, _i64]),
    "bse_c64_prepare": (C.c_int, [_vp, _vp, _i64, _i64, _vp]),
    "bse_chebyshev_filter_c64": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _i64, C.c_int, _dbl, _dbl, _dbl, _vp]),
    "bse_complex_normals": (C.c_int, [_vp, _vp, C.c_uint64, _i64, _i64]),
    "bse_complex_normals_t": (C.c_int, [_vp, _vp, C.c_uint64, _i64, _i64]),
    "bse_symmetrize": (C.c_int, [_vp, _vp, _i64, _i64, C.c_int]),
    "bse_scale_shift": (C.c_int, [_vp, _vp, _i64, _i64, _dbl, _dbl, C.c_int]),
    "bse_eigvalsh": (C.c_int, [_vp, _vp, _i64, _i64, _dp]),
    "bse_zgemm_cn": (C.c_int, [_vp, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64]),
    "bse_zgemm_nn": (C.c_int, [_vp, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64]),
}

# status codes (bse200.h) -> exception classes of the reference (errors.py:8-38)
_STATUS = {
    1: ValidationError,
    2: NumericalError,
    3: IndefiniteError,
    4: RankDeficiencyError,
    5: LanczosBreakdownError,
    6: HermitianRqError,
    7: NumericalError,
}

_lib = None
_lock = threading.Lock()
# Chebyshev-filter product kernels (bse_set_filter_algorithm codes)
_ALGOS = {"4m": 4, "3m": 88, "3m-tma-narrow": 82, "3m-tma-wide": 86, "rs": 90, "rs-tall": 92, "rs-narrow": 94,
          "rs-tall4": 96, "rs-tall4-k32": 97,
          "rs-tall4-k32-split": 98}
# BSE200_FILTER=3m / 4m select the Gauss 3M / plain 4M complex splits for the filter;
# default "rs": the real-split filter (csrc/hop_rs.cuh, 4 n^2 k executed flops per step) for every
# filter product with B != 0 (single GPU and both directions of the 2D grid) and the RR's
# T = S H Q; B = 0 runs "3m" with the B half skipped
_FILTER_CM = _ALGOS[os.environ.get("BSE200_FILTER", "rs").lower()]


def set_filter_algorithm(name: str) -> None:
    """'rs' (default: the real-split planes of csrc/hop_rs.cuh, half the FP64 tensor ops of 4M;
    tile and split-K factor planned per product; fixed unsplit tiles 'rs-tall4-k32' / 'rs-tall4' /
    'rs-tall' / 'rs-narrow', bitwise identical; 'rs-tall4-k32-split' = the first with its K range
    split over 2 CTAs (BSE200_RS_KSPLIT sets the factor)), '3m' (Gauss split, 25% fewer FP64
    tensor ops than 4M, operand sums precomputed once, TMA-fed producer-warp kernel; fixed tiles
    '3m-tma-narrow' / '3m-tma-wide', bitwise identical) or '4m'."""
    global _FILTER_CM
    cm = _ALGOS[name.lower()] if isinstance(name, str) else int(name)
    _FILTER_CM = cm
    for ctx in Context._by_device.values():
        ctx.check(ctx.lib.bse_set_filter_algorithm(ctx.handle, cm))


def filter_algorithm() -> str:
    return {v: k for k, v in _ALGOS.items()}.get(_FILTER_CM, str(_FILTER_CM))


# Chebyshev-filter precision: "c128" (FP64 DMMA, default) or "c64" (FP32-accurate 3xTF32 on the
# tcgen05 tensor cores; configs[4]); the rest of the solve stays complex128
_FILTER_PRECISION = os.environ.get("BSE200_PRECISION", "c128").lower()


def set_filter_precision(name: str) -> None:
    global _FILTER_PRECISION
    if name.lower() not in ("c128", "c64"):
        raise ValueError("filter precision must be 'c128' or 'c64'")
    _FILTER_PRECISION = name.lower()


def filter_precision() -> str:
    return _FILTER_PRECISION


def uses_sum_planes() -> bool:
    return _FILTER_CM in (82, 86, 88) or uses_rs_planes()


def uses_rs_planes() -> bool:
    """real-split filter (codes 90, 92, 94, 96, 97, 98; csrc/hop_rs.cuh); B = 0 products run the 3M kernel (88)"""
    return _FILTER_CM in (90, 92, 94, 96, 97, 98)


def load() -> C.CDLL:
    """Load libbse200.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"bse200 CUDA library not found at {LIB_PATH}; run `python __graft_entry__.py build` "
                    "(no CPU fallback exists)"
                )
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


class Context:
    """One bse_ctx per CUDA device (cuBLAS/cuSOLVER handles + workspace)."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("bse200 needs a CUDA device (B200, sm_100a); none is visible — no CPU fallback")
        self.lib = load()
        self.device = device
        h = _vp()
        st = self.lib.bse_ctx_create(device, C.byref(h))
        if st != 0:
            raise RuntimeError(f"bse_ctx_create failed with status {st}")
        self.handle = h
        self._stream = None
        self.check(self.lib.bse_set_filter_algorithm(h, _FILTER_CM))

    @classmethod
    def get(cls, device: int) -> "Context":
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls(device)
            cls._by_device[device] = ctx
        return ctx

    def bind_stream(self) -> None:
        """Enqueue on torch's current stream of this device."""
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            self.check(self.lib.bse_set_stream(self.handle, _vp(s)))
            self._stream = s

    def check(self, status: int) -> None:
        if status != 0:
            msg = self.lib.bse_last_error(self.handle).decode(errors="replace")
            raise _STATUS.get(status, NumericalError)(msg)

    def call(self, name: str, *args) -> None:
        self.bind_stream()
        self.check(getattr(self.lib, name)(self.handle, *args))

    def set_ham_flags(self, flags: int) -> None:
        if flags != getattr(self, "_ham_flags", None):
            self.check(self.lib.bse_set_hamiltonian_flags(self.handle, flags))
            self._ham_flags = flags

    @property
    def launches(self) -> int:
        return int(self.lib.bse_launch_count(self.handle))


def dptr(t) -> _vp:
    return _vp(None) if t is None else _vp(t.data_ptr())


def planes_fit(nbytes: int, device, reserve: int = 0) -> bool:
    """Whether an optional operand copy of nbytes (the 3M sum planes: +32 m^2 bytes) still leaves
    `reserve` bytes of HBM for the solve's vectors.  Counts memory torch has cached but not used."""
    import torch

    free, _ = torch.cuda.mem_get_info(device)
    cached = torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device)
    return free + cached >= nbytes + reserve + (1 << 30)


def hptr(a) -> _dp:
    return a.ctypes.data_as(_dp)
