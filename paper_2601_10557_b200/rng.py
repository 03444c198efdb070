"""Counter-based random streams, bit-identical to the reference scheme
(bsesolve/rng.py:1-81, docs/FORMATS.md): splitmix64 words, uniforms in
(0, 1], Box-Muller complex normals, column-major matrix fill, tagged child
streams.  Computed on the host with numpy so the start vectors of a solve are
the very same bits the reference draws (GPU libm would differ in the last
ulp and can change a small case's iteration trace).  Above EXACT_LIMIT
(generate.py's policy, n = 100k, where the Hamiltonian itself comes from the
device generator) the start block is drawn on the device: bit-exact words,
Box-Muller within ~1 ulp."""

from __future__ import annotations

import numpy as np

_U64 = np.uint64
_WRAP = (1 << 64) - 1
_STEP, _M1, _M2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _finalize(z):
    z = ((z ^ (z >> 30)) * _M1) & _WRAP
    z = ((z ^ (z >> 27)) * _M2) & _WRAP
    return z ^ (z >> 31)


def word(seed: int, counter: int) -> int:
    return _finalize((seed + (counter + 1) * _STEP) & _WRAP)


def substream(seed: int, tag: int) -> int:
    return word(seed & _WRAP, tag)


def _words(seed: int, start: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = _U64(seed & _WRAP) + np.arange(start + 1, start + 1 + count, dtype=_U64) * _U64(_STEP)
        for shift, mul in ((30, _M1), (27, _M2)):
            z ^= z >> _U64(shift)
            z *= _U64(mul)
        z ^= z >> _U64(31)
    return z


def uniforms(seed: int, start: int, count: int) -> np.ndarray:
    return ((_words(seed, start, count) >> _U64(11)).astype(np.float64) + 1.0) * 2.0**-53


def _normals_serial(seed: int, count: int, start_index: int) -> np.ndarray:
    u = uniforms(seed, 2 * start_index, 2 * count).reshape(count, 2)
    radius = np.sqrt(-2.0 * np.log(u[:, 0]))
    angle = 2.0 * np.pi * u[:, 1]
    return radius * np.cos(angle) + 1j * (radius * np.sin(angle))


_PARALLEL_MIN = 1 << 20
_CHUNK = 1 << 16  # normals per task: the ~10 temporaries of one task stay in L2


def complex_normals(seed: int, count: int, start_index: int = 0, threads: int | None = None) -> np.ndarray:
    """Normals start_index .. start_index+count-1.  Large draws are split into
    cache-sized counter ranges computed on all host cores (numpy ufuncs release
    the GIL); the stream is counter based, so the bits do not depend on the
    split (tests/test_lib_cpu.py checks this)."""
    if count < _PARALLEL_MIN:
        return _normals_serial(seed, count, start_index)
    import os
    from concurrent.futures import ThreadPoolExecutor

    nt = threads or min(64, os.cpu_count() or 1)
    out = np.empty(count, dtype=np.complex128)

    def work(a):
        b = min(a + _CHUNK, count)
        out[a:b] = _normals_serial(seed, b - a, start_index + a)

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(work, range(0, count, _CHUNK)))
    return out


def complex_normals_segments(seed: int, starts, length: int, threads: int | None = None) -> np.ndarray:
    """Row r = normals starts[r] .. starts[r] + length - 1 (equal-length contiguous counter ranges,
    e.g. a row block of a column-major matrix): bit-identical to complex_normals there, computed
    range by range on all host cores (no per-element index arithmetic)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    starts = [int(x) for x in np.ravel(starts)]
    out = np.empty((len(starts), length), dtype=np.complex128)
    if not starts or not length:
        return out
    per = max(1, _CHUNK // length)  # segments per task: ~_CHUNK normals of work each

    def work(a):
        for r in range(a, min(a + per, len(starts))):
            out[r] = _normals_serial(seed, length, starts[r])

    nt = threads or min(64, os.cpu_count() or 1)
    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(work, range(0, len(starts), per)))
    return out


def _normals_at(seed: int, index: np.ndarray) -> np.ndarray:
    """Normals with arbitrary (int64) indices: the same counter arithmetic element by element."""
    ctr = np.empty(2 * index.size, dtype=_U64)
    ctr[0::2] = 2 * index.astype(_U64) + _U64(1)  # word counter c -> state seed + (c + 1) * step
    ctr[1::2] = 2 * index.astype(_U64) + _U64(2)
    with np.errstate(over="ignore"):
        z = _U64(seed & _WRAP) + ctr * _U64(_STEP)
        for shift, mul in ((30, _M1), (27, _M2)):
            z ^= z >> _U64(shift)
            z *= _U64(mul)
        z ^= z >> _U64(31)
    u = (((z >> _U64(11)).astype(np.float64) + 1.0) * 2.0**-53).reshape(index.size, 2)
    radius = np.sqrt(-2.0 * np.log(u[:, 0]))
    angle = 2.0 * np.pi * u[:, 1]
    return radius * np.cos(angle) + 1j * (radius * np.sin(angle))


def complex_normals_at(seed: int, index, threads: int | None = None) -> np.ndarray:
    """Normals #index (any shape), bit-identical to complex_normals at those positions; threaded."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    idx = np.ascontiguousarray(index, dtype=np.int64)
    flat = idx.reshape(-1)
    out = np.empty(flat.size, dtype=np.complex128)
    nt = max(1, min(threads or min(32, os.cpu_count() or 1), flat.size // 65536 + 1))
    edges = np.linspace(0, flat.size, nt + 1).astype(np.int64)

    def work(i):
        a, b = int(edges[i]), int(edges[i + 1])
        out[a:b] = _normals_at(seed, flat[a:b])

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(work, range(nt)))
    return out.reshape(idx.shape)


def device_complex_normal_matrix(seed: int, rows: int, cols: int, device):
    """complex_normal_matrix drawn on the device (bse_complex_normals): column-major rows x cols."""
    import ctypes

    from . import _lib
    from .hamiltonian import colmajor_empty

    out = colmajor_empty(rows, cols, device)
    if rows * cols:
        _lib.Context.get(out.device.index).call("bse_complex_normals", _lib.dptr(out), ctypes.c_uint64(seed), 0,
                                                rows * cols)
    return out


def complex_normal_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    return complex_normals(seed, rows * cols).reshape((cols, rows)).T
