"""CPU check of the algebra behind the real-split filter (csrc/hop_rs.cuh) against the oracle's
apply_h (hamiltonian.py:132-151 restated in oracle/bse_oracle.py::h_times): the folded basis
x = X1 + X2, y = X1 - X2, the four real planes, the filter recurrence run in the folded basis, and
the 2D-tile identities the grid relies on (partial products of folded blocks sum to the folded
product; the transposed tile's planes).  No GPU: this pins the formulation, the GPU tests pin the
kernels (tests/test_gpu_parity.py::test_filter_rs_matches_3m_and_tiles_bitwise)."""
import numpy as np

from conftest import golden_ham
from oracle import bse_oracle as o


def planes(a, b):
    return a.imag + b.imag, a.real - b.real, a.real + b.real, a.imag - b.imag  # Z, V, U, W


def rs_apply(z, v, u, w, x, y):
    return 1j * (z @ x) + v @ y, u @ x + 1j * (w @ y)


def test_folded_operator_matches_apply_h():
    for m, seed in ((16, 5), (64, 21), (8, 11)):
        a, b = golden_ham(m, seed)
        rng = np.random.default_rng(seed)
        X = rng.standard_normal((2 * m, 7)) + 1j * rng.standard_normal((2 * m, 7))
        hx = o.h_times(a, b, X)
        xo, yo = rs_apply(*planes(a, b), X[:m] + X[m:], X[:m] - X[m:])
        scale = np.abs(hx).max()
        assert np.abs(xo - (hx[:m] + hx[m:])).max() <= 1e-13 * scale
        assert np.abs(yo - (hx[:m] - hx[m:])).max() <= 1e-13 * scale


def test_filter_in_folded_basis_matches_oracle_filter():
    a, b = golden_ham(64, 21)
    m = a.shape[0]
    rng = np.random.default_rng(3)
    V = rng.standard_normal((2 * m, 5)) + 1j * rng.standard_normal((2 * m, 5))
    deg, c, e, s = 10, 300.0, 250.0, -600.0
    ref = o.cheb_filter(a, b, V, deg, c, e, s)
    z, v, u, w = planes(a, b)

    def step(Y):  # H Y - c Y in the folded basis (the shift commutes with the fold)
        xo, yo = rs_apply(z, v, u, w, Y[:m], Y[m:])
        return np.vstack([xo, yo]) - c * Y

    F = np.vstack([V[:m] + V[m:], V[:m] - V[m:]])
    s1 = e / (s - c)
    sig = s1
    prev, cur = F, (s1 / e) * step(F)
    for _ in range(2, deg + 1):
        sn = 1.0 / (2.0 / s1 - sig)
        prev, cur = cur, (2.0 * sn / e) * step(cur) - (sig * sn) * prev
        sig = sn
    out = np.vstack([(cur[:m] + cur[m:]) / 2, (cur[:m] - cur[m:]) / 2])
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


def test_tile_partials_and_transposed_planes():
    """2 x 2 grid: the folded partial products of the forward tiles sum to the folded product over
    the row communicator, and the planes of the transposed tile (A_JI, B_JI) are
    (-W_IJ^T, V_IJ^T, U_IJ^T, -Z_IJ^T), i.e. the grid needs no data beyond its two tiles."""
    a, b = golden_ham(64, 21)
    m = a.shape[0]
    rng = np.random.default_rng(4)
    X = rng.standard_normal((2 * m, 3)) + 1j * rng.standard_normal((2 * m, 3))
    hx = o.h_times(a, b, X)
    x, y = X[:m] + X[m:], X[:m] - X[m:]
    edges = [0, 29, m]  # ragged split of the m index space
    for i in range(2):
        r0, r1 = edges[i], edges[i + 1]
        acc_x = np.zeros((r1 - r0, 3), complex)
        acc_y = np.zeros((r1 - r0, 3), complex)
        for j in range(2):
            c0, c1 = edges[j], edges[j + 1]
            pz, pv, pu, pw = planes(a[r0:r1, c0:c1], b[r0:r1, c0:c1])
            px, py = rs_apply(pz, pv, pu, pw, x[c0:c1], y[c0:c1])
            acc_x += px
            acc_y += py
            tz, tv, tu, tw = planes(a[c0:c1, r0:r1], b[c0:c1, r0:r1])
            np.testing.assert_array_equal(tz, -pw.T)
            np.testing.assert_array_equal(tv, pv.T)
            np.testing.assert_array_equal(tu, pu.T)
            np.testing.assert_array_equal(tw, -pz.T)
        scale = np.abs(hx).max()
        assert np.abs(acc_x - (hx[r0:r1] + hx[m + r0:m + r1])).max() <= 1e-13 * scale
        assert np.abs(acc_y - (hx[r0:r1] - hx[m + r0:m + r1])).max() <= 1e-13 * scale
