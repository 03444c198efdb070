"""CPU-side checks of the C ABI boundary: the library loads without a GPU and
exports every symbol include/bse200.h declares; the host logic that needs no
device (config validation, rng, locking, cutoff update) matches the reference."""
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_2601_10557_b200 import _lib
    from paper_2601_10557_b200.build import build_library

    build_library()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    header = (ROOT / "include" / "bse200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(bse_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert b"sm_100a" in _lib.load().bse_version()


def test_sass_has_dmma_and_no_cpu_path():
    import shutil
    import subprocess
    from paper_2601_10557_b200 import _lib

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "LDGSTS" in sass  # cp.async staging (the barrier / mbarrier 3M kernels, zgemm)
    assert "UTMALDG" in sass  # TMA loads (default FP64 filter kernel, complex64 kernel)
    assert "UTCHMMA" in sass  # tcgen05.mma (complex64 filter)
    assert "SYNCS" in sass  # mbarrier pipelines

    # the default filter kernel (real-split planes): DMMA fed by TMA through mbarrier rings
    bodies = [f for f in sass.split("Function : ") if f.startswith("_ZN3bse17hop_rs_tma_kernel")]
    assert bodies
    for body in bodies:
        for op in ("DMMA.8x8x4", "UTMALDG", "SYNCS"):
            assert op in body, op


def test_rng_bit_exact_vs_reference_fixture():
    from paper_2601_10557_b200 import rng

    g = golden("rng.npz")
    assert [rng.word(0, i) for i in range(16)] == [int(w) for w in g["words_seed0"]]
    np.testing.assert_array_equal(rng.complex_normals(12345, 64), g["normals_12345"])
    np.testing.assert_array_equal(rng.complex_normals(rng.substream(0, 3), 257, start_index=5), g["normals_sub03"])
    m = rng.complex_normal_matrix(7, 5, 3)
    np.testing.assert_array_equal(m, g["matrix_7_5_3"])
    assert rng.substream(42, 3) == 0x581CE1FF0E4AE394


def test_solver_config_validation_matches_reference():
    from paper_2601_10557_b200 import SolverConfig, ValidationError

    n = 16
    for bad in [dict(nev=5, nex=5), dict(nev=2, deg=7), dict(nev=0), dict(nev=2, tol=-1.0),
                dict(nev=2, rr_variant="x"), dict(nev=2, lanczos_steps=3), dict(nev=2, maxiter=0)]:
        with pytest.raises(ValidationError):
            SolverConfig(**bad).validate(n)
    SolverConfig(nev=4).validate(n)
    assert SolverConfig(nev=4).nevex == 8 and SolverConfig(nev=4, nex=0).nevex == 4


def test_lock_converged_prefix_window():
    from paper_2601_10557_b200 import RitzSet, lock_converged

    r = RitzSet(values=np.arange(6.0), vectors=None, residual_norms=np.array([1e-9, 1e-9, 1.0, 1e-9, 1e-9, 1e-9]))
    new, act = lock_converged(r, 1e-8, nev=10)
    assert list(new) == [0, 1] and list(act) == [2, 3, 4, 5]
    new, act = lock_converged(r, 1e-8, nev=1)
    assert list(new) == [0]
    r.residual_norms = np.full(6, 1e-9)
    new, _ = lock_converged(r, 1e-8, nev=4)
    assert list(new) == [0, 1, 2, 3]
    r.residual_norms = np.array([2.0, 1e-9])
    new, _ = lock_converged(RitzSet(np.arange(2.0), None, np.array([2.0, 1e-9])), 1e-8, nev=3)
    assert new.size == 0


def test_update_cutoff_and_filter_config():
    from paper_2601_10557_b200 import FilterConfig, SpectralBounds, ValidationError, update_cutoff, scalar_filter_value

    b = SpectralBounds(mu_1=-10.0, mu_nevex=-5.0, mu_n=10.0, steps=4, ritz_values=np.zeros(1), ritz_weights=np.zeros(1))
    assert update_cutoff(b, [-7.0, -6.0]).mu_nevex == -6.0
    assert update_cutoff(b, [-20.0]).mu_nevex == -10.0
    assert update_cutoff(b, [11.0]).mu_nevex == -5.0
    with pytest.raises(ValidationError):
        update_cutoff(b, [])
    with pytest.raises(ValidationError):
        FilterConfig(degree=7, center=0.0, half_width=1.0, scale_ref=-2.0)
    cfg = FilterConfig.from_bounds(b, 16)
    assert scalar_filter_value(cfg.scale_ref, cfg) == pytest.approx(1.0, abs=1e-9)
    from oracle import bse_oracle as o
    for t in np.linspace(-10, 10, 17):
        assert scalar_filter_value(t, cfg) == o.cheb_gain(t, 16, cfg.center, cfg.half_width, cfg.scale_ref)


def test_hamiltonian_validation_on_host():
    from paper_2601_10557_b200 import BseHamiltonian, ValidationError

    with pytest.raises(ValidationError):
        BseHamiltonian(np.array([[1.0, 2.0], [0.0, 1.0]]), np.zeros((2, 2)))
    with pytest.raises(ValidationError):
        BseHamiltonian(np.eye(2), np.zeros((3, 3)))
    with pytest.raises(ValidationError):
        BseHamiltonian(np.array([[np.nan]]), np.zeros((1, 1)))
    a = np.array([[2.0, 1.0 + 1e-14], [1.0, 2.0]], dtype=complex)
    h = BseHamiltonian(a, np.zeros((2, 2)))
    assert np.array_equal(h.a, h.a.conj().T) and h.n == 4


def test_threaded_rng_is_bit_identical():
    from paper_2601_10557_b200 import rng

    count = (1 << 20) + 12345
    ref = rng._normals_serial(99, count, 7)
    for threads in (1, 3, 8):
        np.testing.assert_array_equal(rng.complex_normals(99, count, start_index=7, threads=threads), ref)


def test_indexed_rng_matches_stream():
    from paper_2601_10557_b200 import rng

    full = rng.complex_normal_matrix(rng.substream(0, 3), 40, 7)
    rows = np.r_[3:9, 23:29]
    idx = np.arange(7)[:, None] * 40 + rows[None, :]
    got = rng.complex_normals_at(rng.substream(0, 3), idx, threads=3)
    np.testing.assert_array_equal(got, full[rows].T)
