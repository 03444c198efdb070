"""pytest plugin: run the REFERENCE's own test files against the drop-in.  TEST INFRASTRUCTURE.

Loaded with ``-p dropin_plugin`` by tests/ref_compat/test_reference_suite.py, which points pytest
at the reference's test files (a copy under baseline/_ref/ref_tests, made by
tools/install_reference.sh together with the unmodified reference package in baseline/_ref).

Before the test modules import ``bsesolve``, the solve-path names of the reference package (the
ones SURVEY.md §8(a) puts on the hot path: solve, the filter, the orthonormalisation, the
projections, residuals, locking, bounds, apply_h, is_definite, complete_spectrum,
mirror_largest) are replaced by adapters onto ``paper_2601_10557_b200``.  Dense helpers the tests
use as oracles (generate, materialize, direct_solve_definite, diagnostics, dual_basis_explicit,
scalar_filter_value, rho_sh) stay the reference's own.  The adapters only translate types: the
reference's dataclasses in, ours to the kernels, the reference's dataclasses and exception
classes out.
"""

from __future__ import annotations

import dataclasses
import functools
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
for p in (ROOT / "baseline" / "_ref", ROOT):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

import bsesolve as ref  # noqa: E402  (the unmodified reference package in baseline/_ref)
import bsesolve.chebyshev  # noqa: E402,F401
import bsesolve.hamiltonian  # noqa: E402,F401
import bsesolve.lanczos  # noqa: E402,F401
import bsesolve.ortho  # noqa: E402,F401
import bsesolve.rayleigh_ritz  # noqa: E402,F401
import bsesolve.solver  # noqa: E402,F401

import paper_2601_10557_b200 as ours  # noqa: E402

_HAMS: dict[int, tuple] = {}


def _ham(h):
    """reference BseHamiltonian -> ours (cached per object; definiteness kept in sync)."""
    hit = _HAMS.get(id(h))
    if hit is not None and hit[0] is h:
        o = hit[1]
    else:
        o = ours.BseHamiltonian(h.a, h.b)
        _HAMS[id(h)] = (h, o)
    if h.definiteness.name != "UNKNOWN":
        o.definiteness = ours.Definiteness[h.definiteness.name]
    return o


def _same_fields(cls, obj, **over):
    kw = {f.name: getattr(obj, f.name) for f in dataclasses.fields(cls) if f.name not in over and hasattr(obj, f.name)}
    kw.update(over)
    return cls(**kw)


def to_ours(x):
    if isinstance(x, ref.BseHamiltonian):
        return _ham(x)
    if isinstance(x, ref.FilterConfig):
        return _same_fields(ours.FilterConfig, x)
    if isinstance(x, ref.SolverConfig):
        return _same_fields(ours.SolverConfig, x)
    if isinstance(x, ref.SpectralBounds):
        return _same_fields(ours.SpectralBounds, x)
    if isinstance(x, ref.SolveResult):
        return _same_fields(ours.SolveResult, x, trace=[_same_fields(ours.TraceRecord, t) for t in x.trace],
                            bounds=to_ours(x.bounds))
    return x


def to_ref(x):
    if isinstance(x, tuple):
        return tuple(to_ref(y) for y in x)
    if isinstance(x, ours.SolveResult):
        led = ref.PhaseLedger()
        led.flops.update(x.ledger.flops)
        led.seconds.update(x.ledger.seconds)
        return _same_fields(ref.SolveResult, x, trace=[_same_fields(ref.TraceRecord, t) for t in x.trace],
                            bounds=to_ref(x.bounds), ledger=led)
    if isinstance(x, ours.SpectralBounds):
        return _same_fields(ref.SpectralBounds, x)
    if isinstance(x, ours.RitzSet):
        return _same_fields(ref.RitzSet, x)
    if isinstance(x, ours.ReducedProblem):
        return _same_fields(ref.rayleigh_ritz.ReducedProblem, x)
    if isinstance(x, ours.SearchSpace):
        return _same_fields(ref.ortho.SearchSpace, x)
    if isinstance(x, ours.CompletedSpectrum):
        return _same_fields(ref.solver.CompletedSpectrum, x)
    if isinstance(x, ours.Definiteness):
        return ref.Definiteness[x.name]
    return x


def adapt(fn, sync_ham: bool = False):
    @functools.wraps(fn)
    def call(*args, **kw):
        oargs = [to_ours(a) for a in args]
        okw = {k: to_ours(v) for k, v in kw.items()}
        try:
            out = fn(*oargs, **okw)
        except ours.BseSolveError as exc:
            raise getattr(ref.errors, type(exc).__name__)(str(exc)) from exc
        finally:
            if sync_ham:
                for a, o in zip(args, oargs):
                    if isinstance(a, ref.BseHamiltonian) and o.definiteness.name != "UNKNOWN":
                        a.definiteness = ref.Definiteness[o.definiteness.name]
        return to_ref(out)

    call.__dropin__ = True
    return call


# (name, modules that hold it) -- every binding the tests or the reference's own internals reach
PATCHES = {
    "solve": ("bsesolve", "bsesolve.solver"),
    "complete_spectrum": ("bsesolve", "bsesolve.solver"),
    "mirror_largest": ("bsesolve", "bsesolve.solver"),
    "chebyshev_filter": ("bsesolve", "bsesolve.chebyshev"),
    "estimate_bounds": ("bsesolve", "bsesolve.lanczos"),
    "update_cutoff": ("bsesolve", "bsesolve.lanczos"),
    "s_orthonormalize": ("bsesolve", "bsesolve.ortho"),
    "cholqr_with_fallback": ("bsesolve", "bsesolve.ortho"),
    "fix_column_phases": ("bsesolve", "bsesolve.ortho"),
    "build_hermitian_rq": ("bsesolve", "bsesolve.rayleigh_ritz"),
    "build_backup_rq": ("bsesolve", "bsesolve.rayleigh_ritz"),
    "residuals": ("bsesolve", "bsesolve.rayleigh_ritz"),
    "lock_converged": ("bsesolve", "bsesolve.rayleigh_ritz"),
    "apply_h": ("bsesolve", "bsesolve.hamiltonian"),
    "apply_h_via_adjoint": ("bsesolve", "bsesolve.hamiltonian"),
    "is_definite": ("bsesolve", "bsesolve.hamiltonian"),
}


def install() -> None:
    for name, mods in PATCHES.items():
        fn = adapt(getattr(ours, name), sync_ham=name in ("is_definite", "solve"))
        for mod in mods:
            setattr(sys.modules[mod], name, fn)


def pytest_configure(config):
    install()
