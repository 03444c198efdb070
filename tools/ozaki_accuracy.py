"""Accuracy study (design note): integer-slice
(Ozaki-I) emulation of the complex filter product A X vs native FP64, on blocks built like the
reference generator (A = C C^H + I, B = 0.5 lambda_min(A) / sigma_max(B0) B0, generate.py:60-83).
Exact reference in long double.  CPU only: python tools/ozaki_accuracy.py"""
import numpy as np


def make_blocks(m, seed=0):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    a = c @ c.conj().T + np.eye(m)
    d = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    b0 = (d + d.T) / 2
    b = 0.5 * np.linalg.eigvalsh(a)[0] / np.linalg.norm(b0, 2) * b0
    return a, b

def slices(v, s, axis):
    """rows (axis=1 -> per-row scale) of complex v: integer digits d_1..d_s in [-64,64], scale 2^e."""
    mx = np.maximum(np.abs(v.real).max(axis=axis, keepdims=True), np.abs(v.imag).max(axis=axis, keepdims=True))
    e = np.ceil(np.log2(np.where(mx > 0, mx, 1.0)))
    r_re, r_im = v.real / 2.0**e, v.imag / 2.0**e          # |r| <= 1
    out = []
    for i in range(s):
        dr, di = np.round(r_re * 64), np.round(r_im * 64)
        out.append((dr, di))
        r_re, r_im = r_re * 64 - dr, r_im * 64 - di          # |r| <= 0.5 -> next digit in [-32,32]*2
        r_re, r_im = r_re * 2, r_im * 2
    return out, e

def ozaki(a, x, s):
    da, ea = slices(a, s, 1)
    dx, ex = slices(x, s, 0)
    yr = np.zeros((a.shape[0], x.shape[1])); yi = np.zeros_like(yr)
    # digit i carries weight 2^-(6 + 7(i-1)) ... (first 64*r -> weight 2^-6, then x128 per level)
    for i in range(s):
        for j in range(s - i):
            w = 2.0 ** (-(6 + 7 * i) - (6 + 7 * j))
            ar, ai = da[i]; xr, xi = dx[j]
            yr += w * (ar @ xr - ai @ xi)   # exact in int (checked by magnitude) then one rounding
            yi += w * (ar @ xi + ai @ xr)
    return (yr + 1j * yi) * 2.0**ea * 2.0**ex

def exact(a, x):
    al = a.astype(np.clongdouble); xl = x.astype(np.clongdouble)
    return al @ xl

for m in (1000, 2000):
    a, b = make_blocks(m)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((m, 8)) + 1j * rng.standard_normal((m, 8))
    x[:, 1] *= 1e-3; x[:, 2] *= np.logspace(0, -6, m)  # column scales and a graded column
    for name, mat in (("A", a), ("B", b)):
        ref = exact(mat, x)
        scale = (np.abs(mat).astype(np.longdouble) @ np.abs(x).astype(np.longdouble))
        e64 = np.abs((mat @ x) - ref) / scale
        line = [f"m={m} {name}: fp64 max {float(e64.max()):.2e} med {float(np.median(e64)):.2e}"]
        for s in (6, 7, 8):
            eo = np.abs(ozaki(mat, x, s) - ref) / scale
            line.append(f"s={s}: max {float(eo.max()):.2e} med {float(np.median(eo)):.2e}")
        print(" | ".join(line), flush=True)
