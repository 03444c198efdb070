"""CPU oracle: a numpy restatement of the reference pseudo-hermitian ChASE solve.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2601_10557_b200`` imports this
module; it is used by ``tests/``, ``__graft_entry__.smoke()`` (as the checker)
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs (as the CPU
baseline).  The product path never routes through it.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this restatement
against fixtures produced by the reference package itself
(``oracle/make_golden.py`` imports ``bsesolve`` from /root/reference in the
build container and writes ``tests/golden/*.npz``).

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/bsesolve/).  The arithmetic is complex128 numpy /
scipy (OpenBLAS + LAPACK), exactly the calls the reference makes, so on one
machine the oracle reproduces the reference bit-for-bit where the reference
is deterministic.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

# ----------------------------------------------------------------------------
# rng.py:37-81  splitmix64 counter streams + Box-Muller complex normals
# ----------------------------------------------------------------------------
M64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
MIX_A = 0xBF58476D1CE4E5B9
MIX_B = 0x94D049BB133111EB


def sm64(seed: int, ctr: int) -> int:
    """rng.py:37-42 (scalar normative definition)."""
    z = (seed + (ctr + 1) * GOLDEN_GAMMA) & M64
    z = ((z ^ (z >> 30)) * MIX_A) & M64
    z = ((z ^ (z >> 27)) * MIX_B) & M64
    return z ^ (z >> 31)


def child_seed(seed: int, tag: int) -> int:
    """rng.py:45-47."""
    return sm64(seed & M64, tag)


def sm64_block(seed: int, first: int, count: int) -> np.ndarray:
    """rng.py:50-60 vectorised words for counters first..first+count-1."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & M64) + np.arange(first + 1, first + count + 1, dtype=np.uint64) * np.uint64(GOLDEN_GAMMA)
        z ^= z >> np.uint64(30)
        z *= np.uint64(MIX_A)
        z ^= z >> np.uint64(27)
        z *= np.uint64(MIX_B)
        z ^= z >> np.uint64(31)
    return z


def gauss_c(seed: int, count: int, first: int = 0) -> np.ndarray:
    """rng.py:63-75: uniforms in (0,1] then Box-Muller on counter pairs."""
    u = ((sm64_block(seed, 2 * first, 2 * count) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
    rad = np.sqrt(-2.0 * np.log(u[0::2]))
    phi = 2.0 * np.pi * u[1::2]
    return rad * np.cos(phi) + 1j * (rad * np.sin(phi))


def gauss_c_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    """rng.py:78-81 column-major fill."""
    return np.asfortranarray(gauss_c(seed, rows * cols).reshape((rows, cols), order="F"))


# ----------------------------------------------------------------------------
# hamiltonian.py / generate.py
# ----------------------------------------------------------------------------
def h_times(a: np.ndarray, b: np.ndarray, x: np.ndarray) -> np.ndarray:
    """hamiltonian.py:132-151: H x = [A x1 + B x2; -conj(A conj x2 + B conj x1)]."""
    m = a.shape[0]
    x1, x2 = x[:m], x[m:]
    top = a @ x1 + b @ x2
    bot = -np.conj(a @ np.conj(x2) + b @ np.conj(x1))
    return np.concatenate([top, bot], axis=0)


def h_times_adjoint(a: np.ndarray, b: np.ndarray, x: np.ndarray) -> np.ndarray:
    """hamiltonian.py:154-176: H x computed as S (H* (S x)) -- the form the
    reference's filter uses on odd steps (chebyshev.py:62-65).  Same bits as
    h_times on one device up to roundoff; kept for timing fidelity."""
    m = a.shape[0]
    y1, y2 = x[:m], -x[m:]
    up = a @ y1 - b @ y2
    low = np.conj(b @ np.conj(y1) - a @ np.conj(y2))
    return np.concatenate([up, -low], axis=0)


def s_flip(x: np.ndarray) -> np.ndarray:
    """hamiltonian.py:104-111."""
    y = np.array(x, dtype=np.complex128, copy=True)
    y[y.shape[0] // 2:] *= -1.0
    return y


def dense_h(a, b):
    """hamiltonian.py:179-183."""
    return np.block([[a, b], [-np.conj(b), -np.conj(a)]])


def dense_sh(a, b):
    """hamiltonian.py:186-190."""
    return np.block([[a, b], [np.conj(b), np.conj(a)]])


def sh_is_definite(a, b) -> bool:
    """hamiltonian.py:208-218."""
    try:
        sla.cholesky(dense_sh(a, b), lower=True)
    except sla.LinAlgError:
        return False
    return True


def make_instance(m: int, seed: int, alpha: float = 1.0, coupling: float = 0.5):
    """generate.py:60-83; returns (A, B, scale_info)."""
    cmat = gauss_c_matrix(child_seed(seed, 0), m, m)
    a = cmat @ cmat.conj().T + alpha * np.eye(m)
    a = (a + a.conj().T) / 2.0
    info = {}
    if coupling == 0.0:
        b = np.zeros((m, m), dtype=np.complex128)
    else:
        d = gauss_c_matrix(child_seed(seed, 1), m, m)
        b0 = (d + d.T) / 2.0
        bnorm = sla.svdvals(b0)[0]
        lmin = float(sla.eigvalsh(a)[0])
        info = {"b0_norm": float(bnorm), "lambda_min_a": lmin}
        b = (coupling * lmin / bnorm) * b0
    return np.asfortranarray(a), np.asfortranarray(b), info


# ----------------------------------------------------------------------------
# lanczos.py:53-181
# ----------------------------------------------------------------------------
@dataclass
class Bounds:
    mu_1: float
    mu_nevex: float
    mu_n: float
    steps: int
    ritz_values: np.ndarray
    ritz_weights: np.ndarray


def _lanczos_sweep(a, b, start, steps, flops):
    """lanczos.py:53-88 (S-inner-product Lanczos, one H product per step)."""
    hv = h_times(a, b, start)
    flops[0] += 8.0 * (2 * a.shape[0]) ** 2
    nrm2 = np.real(np.vdot(s_flip(hv), start))
    if nrm2 <= 0:
        raise ArithmeticError("indefinite")
    sc = np.sqrt(nrm2)
    q, z = start / sc, hv / sc
    q_old = np.zeros_like(start)
    beta_old = 0.0
    al, be = [], []
    for j in range(steps):
        al.append(float(np.real(np.vdot(s_flip(z), z))))
        if j == steps - 1:
            break
        w = z - al[-1] * q - beta_old * q_old
        g = h_times(a, b, w)
        flops[0] += 8.0 * (2 * a.shape[0]) ** 2
        b2 = float(np.real(np.vdot(s_flip(g), w)))
        ref = max(1.0, max(abs(t) for t in al), beta_old)
        if b2 <= (1e-14 * ref) ** 2:
            break
        beta = np.sqrt(b2)
        be.append(beta)
        q_old, q = q, w / beta
        z = g / beta
        beta_old = beta
    return np.array(al), np.array(be), len(al) < steps


def lanczos_bounds(a, b, nevex, steps, seed, flops):
    """lanczos.py:91-142 + _density_cutoff :145-164."""
    n = 2 * a.shape[0]
    al = be = np.empty(0)
    for attempt in range(4):  # MAX_RESTARTS = 3
        start = gauss_c(child_seed(seed, attempt), n)
        al, be, early = _lanczos_sweep(a, b, start, steps, flops)
        if not early or len(al) >= min(4, steps):
            break
    if len(al) < min(4, steps):
        raise ArithmeticError("lanczos breakdown")
    if len(al) % 2:
        al = al[:-1]
        be = be[: len(al) - 1]
    theta, y = sla.eigh_tridiagonal(al, be)
    wts = y[0, :] ** 2
    mu1 = float(theta[0]) - 0.01 * abs(float(theta[0]))
    neg = theta < 0
    if not neg.any():
        cut = 0.0
    else:
        csum = np.cumsum(wts[neg])
        hit = np.nonzero(csum >= nevex / n)[0]
        j = int(hit[0]) if hit.size else int(neg.sum()) - 1
        cut = float((theta[j] + theta[j + 1]) / 2.0) if j + 1 < theta.shape[0] else float(theta[j])
    cut = float(min(max(cut, mu1), -mu1))
    return Bounds(mu1, cut, -mu1, len(al), theta, wts)


# ----------------------------------------------------------------------------
# chebyshev.py:51-89
# ----------------------------------------------------------------------------
def cheb_filter(a, b, v, deg, c, e, s, flops=None):
    """chebyshev.py:51-75 (plain product every step; the adjoint form is
    bitwise-equal on one device, hamiltonian.py:154-176)."""
    n = 2 * a.shape[0]
    k = v.shape[1]
    sig1 = e / (s - c)
    sig = sig1
    y_old = v
    y = (h_times(a, b, v) - c * v) * (sig1 / e)
    for _ in range(2, deg + 1):
        sn = 1.0 / (2.0 / sig1 - sig)
        y_new = (2.0 * sn / e) * (h_times(a, b, y) - c * y) - (sig * sn) * y_old
        y_old, y, sig = y, y_new, sn
    if flops is not None:
        flops[0] += deg * 8.0 * n * n * k
    return y


def cheb_gain(t, deg, c, e, s):
    """chebyshev.py:78-89."""
    sig1 = e / (s - c)
    sig = sig1
    y_old, y = 1.0, (t - c) * (sig1 / e)
    for _ in range(2, deg + 1):
        sn = 1.0 / (2.0 / sig1 - sig)
        y_old, y, sig = y, (2.0 * sn / e) * (t - c) * y - (sig * sn) * y_old, sn
    return y


# ----------------------------------------------------------------------------
# ortho.py:70-158
# ----------------------------------------------------------------------------
def phase_fix(q):
    """ortho.py:70-82: first entry with |q| >= 1e-8 max|q| made real positive."""
    out = q.copy()
    for j in range(out.shape[1]):
        mag = np.abs(out[:, j])
        top = mag.max()
        if top == 0.0:
            continue
        p = out[np.nonzero(mag >= 1e-8 * top)[0][0], j]
        out[:, j] *= np.conj(p) / np.abs(p)
    return out


def cholqr2(x, flops=None):
    """ortho.py:96-129: CholQR twice, accept if max|Q*Q-I| <= 1e-8, else
    Householder with rank test 1e-10."""
    n, k = x.shape
    if k > n:
        raise ArithmeticError("rank")
    if flops is not None:
        flops[0] += 2 * (8.0 * n * k * k + 4.0 * n * k * k)
    q, how = x, "cholqr"
    for _ in range(2):
        g = q.conj().T @ q
        g = (g + g.conj().T) / 2.0
        try:
            r = sla.cholesky(g, lower=False)
            q = sla.solve_triangular(r, q.T, trans="T", lower=False).T
        except sla.LinAlgError:
            how = "householder"
            break
    if how == "cholqr" and not np.abs(q.conj().T @ q - np.eye(k)).max() <= 1e-8:
        how = "householder"
    if how == "householder":
        q, r = np.linalg.qr(x)
        d = np.abs(np.diag(r))
        if d.max() == 0.0 or d.min() <= 1e-10 * d.max():
            raise ArithmeticError("rank")
    return phase_fix(q), how


def s_ortho(v, locked, flops=None):
    """ortho.py:132-158: project out span(S Y_locked), then CholQR2."""
    if locked.shape[1]:
        basis, _ = np.linalg.qr(s_flip(locked))
        v = v - basis @ (basis.conj().T @ v)
        if flops is not None:
            flops[0] += 16.0 * v.shape[0] * basis.shape[1] * v.shape[1]
    q, how = cholqr2(v, flops)
    return q, how


# ----------------------------------------------------------------------------
# rayleigh_ritz.py:85-214, direct.py:86-116
# ----------------------------------------------------------------------------
class RqFailure(ArithmeticError):
    pass


def _m_matrix(q):
    """rayleigh_ritz.py:90-95."""
    q2 = q[q.shape[0] // 2:]
    mm = np.eye(q.shape[1]) - 2.0 * (q2.conj().T @ q2)
    return (mm + mm.conj().T) / 2.0


def rr_hermitian(a, b, q, flops=None):
    """rayleigh_ritz.py:98-143 (Alg. 2)."""
    n, k = q.shape
    t = s_flip(h_times(a, b, q))
    w = q.conj().T @ t
    w = (w + w.conj().T) / 2.0
    mm = _m_matrix(q)
    lam_min_m = float(np.abs(np.linalg.eigvalsh(mm)).min())
    if lam_min_m < 1e-8:
        raise RqFailure("M singular")
    try:
        ell = sla.cholesky(w, lower=True)
    except sla.LinAlgError as exc:
        raise RqFailure("W not definite") from exc
    g = sla.solve_triangular(ell, mm, lower=True)
    g = sla.solve_triangular(ell, g.conj().T, lower=True).conj().T
    g = (g + g.conj().T) / 2.0
    theta, y = np.linalg.eigh((g + g.conj().T) / 2.0)
    if np.abs(theta).min() < np.finfo(float).eps:
        raise RqFailure("theta ~ 0")
    lam = 1.0 / theta
    vec = q @ sla.solve_triangular(ell.conj().T, y, lower=False)
    vec /= np.linalg.norm(vec, axis=0)
    order = np.argsort(lam, kind="stable")
    if flops is not None:
        # apply_h charges 8n^2k to "rr" (hamiltonian.py:148-150) and the RR
        # step charges its own model on top (rayleigh_ritz.py:139)
        flops[0] += 8.0 * n * n * k + 8.0 * n * n * k + 12.0 * n * k * k + 16.0 * k**3
    return lam[order], vec[:, order], lam_min_m


def rr_backup(a, b, q, flops=None):
    """rayleigh_ritz.py:146-179 (Alg. 3) + direct.py:102-116."""
    n, k = q.shape
    t = h_times(a, b, q)
    w = q.conj().T @ t
    mm = _m_matrix(q)
    lam_min_m = float(np.abs(np.linalg.eigvalsh(mm)).min())
    dv = np.real(np.diag(mm)).copy()
    dv[np.abs(dv) <= 1e-12] = 1.0
    g = (q.conj().T @ s_flip(t) - (mm - np.diag(np.diag(mm))) @ w) / dv[:, None]
    vals, y = sla.eig(g)
    o = np.argsort(vals.real, kind="stable")
    vals, y = vals[o], y[:, o]
    lam = vals.real.copy()
    vec = q @ y
    vec /= np.linalg.norm(vec, axis=0)
    order = np.argsort(lam, kind="stable")
    if flops is not None:
        flops[0] += 8.0 * n * n * k + 8.0 * n * n * k + 20.0 * n * k * k + 30.0 * k**3
    return lam[order], vec[:, order], lam_min_m


def residual_norms(a, b, lam, vec):
    """rayleigh_ritz.py:182-190."""
    return np.linalg.norm(h_times(a, b, vec) - vec * lam, axis=0)


def converged_prefix(res, tol, cap, normalizer=1.0):
    """rayleigh_ritz.py:193-214: longest converged prefix, capped."""
    ok = res <= tol * normalizer
    cnt = 0
    while cnt < res.shape[0] and cnt < cap and ok[cnt]:
        cnt += 1
    return cnt, ok


# ----------------------------------------------------------------------------
# solver.py:125-250
# ----------------------------------------------------------------------------
@dataclass
class OracleResult:
    lambdas: np.ndarray
    v: np.ndarray
    residual_norms: np.ndarray
    iterations_used: int
    converged: bool
    trace: list = field(default_factory=list)
    bounds: Bounds | None = None
    flops: dict = field(default_factory=dict)
    backup_events: int = 0


def oracle_solve(a, b, nev, nex=None, deg=20, tol=1e-8, maxiter=25, rr_variant="auto",
                 seed=0, lanczos_steps=24, rel_res=False, seconds=None):
    """solver.py:125-250 outer loop (trace rows: it, locked, k, max_res,
    min_res_unlocked, mu_nevex, variant, lambda_min_m, flops).  ``seconds``
    (a dict) receives per-phase wall seconds like the reference's PhaseLedger
    (metrics.py:11-39, solver.py:157-184)."""
    import time as _time

    sec = seconds if seconds is not None else {}
    clock = [_time.perf_counter()]

    def lap(phase):
        now = _time.perf_counter()
        sec[phase] = sec.get(phase, 0.0) + now - clock[0]
        clock[0] = now

    m = a.shape[0]
    n = 2 * m
    nevex = nev + (nev if nex is None else nex)
    fl = {p: [0.0] for p in ("lanczos", "filter", "ortho", "rr", "residuals")}
    bnd = lanczos_bounds(a, b, nevex, lanczos_steps, child_seed(seed, 2), fl["lanczos"])
    lap("lanczos")
    normalizer = abs(bnd.mu_1) if rel_res else 1.0
    vhat = gauss_c_matrix(child_seed(seed, 3), n, nevex)
    lap("start")
    lk_vals, lk_res = [], []
    lk_y = np.zeros((n, 0), dtype=np.complex128)
    trace, backups, done, it_used = [], 0, False, 0
    cur_cut = bnd.mu_nevex
    lam = vec = res = act = None
    for it in range(1, maxiter + 1):
        it_used = it
        before = sum(v[0] for v in fl.values())
        k = nevex - len(lk_vals)
        c, e = (bnd.mu_n + cur_cut) / 2.0, (bnd.mu_n - cur_cut) / 2.0
        vhat = cheb_filter(a, b, vhat, deg, c, e, bnd.mu_1, fl["filter"])
        lap("filter")
        q_act, _ = s_ortho(vhat, lk_y, fl["ortho"])
        lap("ortho")
        variant = "hermitian"
        if rr_variant == "backup":
            variant = "backup"
            lam, vec, lmm = rr_backup(a, b, q_act, fl["rr"])
        else:
            try:
                lam, vec, lmm = rr_hermitian(a, b, q_act, fl["rr"])
            except RqFailure:
                if rr_variant == "hermitian":
                    raise
                variant = "backup"
                backups += 1
                lam, vec, lmm = rr_backup(a, b, q_act, fl["rr"])
        lap("rr")
        res = residual_norms(a, b, lam, vec)
        lap("residuals")
        fl["residuals"][0] += 8.0 * n * n * vec.shape[1]
        cnt, ok = converged_prefix(res, tol, nev - len(lk_vals), normalizer)
        if cnt:
            lk_y = np.concatenate([lk_y, vec[:, :cnt]], axis=1)
            lk_vals.extend(lam[:cnt])
            lk_res.extend(res[:cnt])
        act = np.arange(cnt, lam.shape[0])
        trace.append(dict(it=it, locked=len(lk_vals), k=k, max_res=float(res.max()),
                          min_res_unlocked=float(res[act].min()) if act.size else 0.0,
                          mu_nevex=cur_cut, variant=variant, lambda_min_m=lmm,
                          flops=sum(v[0] for v in fl.values()) - before))
        if len(lk_vals) >= nev:
            done = True
            break
        vhat = vec[:, act]
        out = lam[act][~ok[act]]
        cand = out if out.size else lam[act]
        cand = np.minimum(cand[cand >= bnd.mu_1], 0.0)
        if cand.size:
            top = float(cand.max())
            if top < bnd.mu_n:
                cur_cut = max(top, bnd.mu_1)
    if done:
        vals, vecs, rr = np.array(lk_vals), lk_y, np.array(lk_res)
    else:
        miss = nev - len(lk_vals)
        vals = np.concatenate([lk_vals, lam[act][:miss]])
        vecs = np.concatenate([lk_y, vec[:, act[:miss]]], axis=1)
        rr = np.concatenate([lk_res, res[act][:miss]])
    o = np.argsort(vals, kind="stable")[:nev]
    return OracleResult(vals[o], vecs[:, o], rr[o], it_used, done, trace, bnd,
                        {p: v[0] for p, v in fl.items()}, backups)


def dense_eigs(a, b):
    """direct.py:43-59: all eigenvalues via the Cholesky reduction (n <= 4096)."""
    sh = dense_sh(a, b)
    ell = sla.cholesky(sh, lower=True)
    red = ell.conj().T @ s_flip(ell)
    red = (red + red.conj().T) / 2.0
    return np.linalg.eigvalsh(red)
