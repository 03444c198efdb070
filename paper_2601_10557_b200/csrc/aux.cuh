// HBM-bound helper kernels: column norms / scaling, phase convention, S flip,
// small k x k fix-ups, deterministic dot products and reductions.
// Every reduction is a fixed-order tree (no atomics): reruns are bitwise equal.
#pragma once
#include "common.cuh"

namespace bse {

constexpr int RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    r = warp_max(r);
  }
  __syncthreads();
  return r;
}

// norms[j] = ||x[:, j]||_2 (one CTA per column)  — np.linalg.norm(axis=0)
__global__ void colnorm_kernel(const zval* __restrict__ x, int64_t ldx, int64_t n, double* __restrict__ norms) {
  __shared__ double sh[32];
  const zval* col = x + (int64_t)blockIdx.x * ldx;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const zval v = col[i];
    s += v.re * v.re + v.im * v.im;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) norms[blockIdx.x] = sqrt(s);
}

// x[:, j] /= norms[j]
__global__ void colscale_inv_kernel(zval* __restrict__ x, int64_t ldx, int64_t n, const double* __restrict__ norms) {
  const double s = norms[blockIdx.y];
  zval* col = x + (int64_t)blockIdx.y * ldx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    zval v = col[i];
    v.re /= s;
    v.im /= s;
    col[i] = v;
  }
}

// ortho.py:70-82: scale column j by conj(p)/|p| where p is the first entry
// with |q| >= 1e-8 * max|q| (columns of zeros untouched).  One CTA per column.
__global__ void phase_fix_kernel(zval* __restrict__ q, int64_t ldq, int64_t n) {
  __shared__ double sh[32];
  __shared__ long long first_sh[32];
  zval* col = q + (int64_t)blockIdx.x * ldq;
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const zval v = col[i];
    mx = fmax(mx, hypot(v.re, v.im));
  }
  mx = block_max(mx, sh);
  if (threadIdx.x == 0) sh[0] = mx;
  __syncthreads();
  mx = sh[0];
  __syncthreads();
  if (mx == 0.0) return;
  const double thr = 1e-8 * mx;
  long long first = n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const zval v = col[i];
    if (hypot(v.re, v.im) >= thr) {
      first = i;
      break;
    }
  }
  // block min
  for (int o = 16; o > 0; o >>= 1) first = min(first, (long long)__shfl_xor_sync(0xffffffffu, first, o));
  if ((threadIdx.x & 31) == 0) first_sh[threadIdx.x >> 5] = first;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long f = first_sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) f = min(f, first_sh[w]);
    first_sh[0] = f;
  }
  __syncthreads();
  const zval p = col[first_sh[0]];
  const double ap = hypot(p.re, p.im);
  const double fr = p.re / ap, fi = -p.im / ap;  // conj(p)/|p|
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const zval v = col[i];
    col[i] = zval{v.re * fr - v.im * fi, v.re * fi + v.im * fr};
  }
}

// y = S x (lower half negated), n = 2m rows, k columns
__global__ void sflip_copy_kernel(const zval* __restrict__ x, int64_t ldx, zval* __restrict__ y, int64_t ldy, int64_t m,
                                  int64_t k) {
  const int64_t total = 2 * m * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx % (2 * m), col = idx / (2 * m);
    zval v = x[col * ldx + row];
    if (row >= m) {
      v.re = -v.re;
      v.im = -v.im;
    }
    y[col * ldy + row] = v;
  }
}

// g <- (g + g^H) / 2 for a k x k matrix (ld = k); one thread per (i, j) with i <= j
// hermitian matrix from its upper triangle (GEMM_UPPER Grams): lower = conj(upper), real diagonal
__global__ void herm_upper_kernel(zval* g, int k) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % k), j = int(idx / k);
    if (i > j) continue;
    const zval a = g[(int64_t)j * k + i];
    if (i == j) {
      g[(int64_t)j * k + i] = zval{a.re, 0.0};
    } else {
      g[(int64_t)i * k + j] = zval{a.re, -a.im};
    }
  }
}

__global__ void hermitize_kernel(zval* g, int k) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % k), j = int(idx / k);
    if (i > j) continue;
    const zval a = g[(int64_t)j * k + i], b = g[(int64_t)i * k + j];
    // (a + conj(b)) / 2 at (i, j); its conjugate at (j, i)
    const zval s{(a.re + b.re) / 2.0, (a.im - b.im) / 2.0};
    g[(int64_t)j * k + i] = s;
    g[(int64_t)i * k + j] = zval{s.re, -s.im};
  }
}

// m <- I - 2 g2 (then hermitized by the caller): rayleigh_ritz.py:90-95
__global__ void form_m_kernel(const zval* __restrict__ g2, zval* __restrict__ mm, int k) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % k), j = int(idx / k);
    const zval v = g2[idx];
    mm[idx] = zval{(i == j ? 1.0 : 0.0) - 2.0 * v.re, -2.0 * v.im};
  }
}

// out = max |g - I| over a k x k matrix: per-CTA maxima, NaN-propagating
__global__ void defect_partial_kernel(const zval* __restrict__ g, int k, double* __restrict__ part) {
  __shared__ double sh[32];
  __shared__ int saw_nan;
  if (threadIdx.x == 0) saw_nan = 0;
  __syncthreads();
  const int64_t total = (int64_t)k * k;
  double mx = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % k), j = int(idx / k);
    zval v = g[idx];
    if (i == j) v.re -= 1.0;
    const double a = hypot(v.re, v.im);
    if (a != a) saw_nan = 1;
    mx = fmax(mx, a);
  }
  mx = block_max(mx, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = saw_nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
}

// single-thread fixed-order max over np partials (NaN wins)
__global__ void max_reduce_kernel(const double* __restrict__ part, int np, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mx = 0.0;
  for (int i = 0; i < np; ++i) {
    const double v = part[i];
    if (v != v) { mx = v; break; }
    mx = fmax(mx, v);
  }
  out[0] = mx;
}

// out[:, j] = in[:, perm[j]] for an r x k matrix (ld_in, ld_out)
__global__ void gather_cols_kernel(const zval* __restrict__ in, int64_t ldi, zval* __restrict__ out, int64_t ldo,
                                   int64_t rows, const int* __restrict__ perm) {
  const zval* src = in + (int64_t)perm[blockIdx.y] * ldi;
  zval* dst = out + (int64_t)blockIdx.y * ldo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// partial[bx] = sum_i sgn_i * conj(x_i) y_i  (sgn = -1 on rows >= m when sflip), real part only
__global__ void sdot_partial_kernel(const zval* __restrict__ x, const zval* __restrict__ y, int64_t n, int64_t m,
                                    int sflip, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const zval a = x[i], b = y[i];
    const double v = a.re * b.re + a.im * b.im;
    s += (sflip && i >= m) ? -v : v;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_reduce_kernel(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[0] = s;
}

// residual partials [nb][k] -> norms[k] (fixed order)
__global__ void resid_finalize_kernel(const double* __restrict__ part, int nb, int k, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * k + j];
  out[j] = sqrt(s);
}

// z = a*x + b*y + c*w  (real coefficients; a pointer may be null when its coefficient is 0)
__global__ void lincomb3_kernel(zval* __restrict__ z, const zval* x, double a, const zval* y, double b, const zval* w,
                                double c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    zval r{0.0, 0.0};
    if (a != 0.0) { const zval v = x[i]; r.re = a * v.re; r.im = a * v.im; }
    if (b != 0.0) { const zval v = y[i]; r.re = __dadd_rn(r.re, __dmul_rn(b, v.re)); r.im = __dadd_rn(r.im, __dmul_rn(b, v.im)); }
    if (c != 0.0) { const zval v = w[i]; r.re = __dadd_rn(r.re, __dmul_rn(c, v.re)); r.im = __dadd_rn(r.im, __dmul_rn(c, v.im)); }
    z[i] = r;
  }
}

// materialise S H = [[A, B], [conj B, conj A]] (n x n, ld = n) from [A | B]
__global__ void materialize_sh_kernel(const zval* __restrict__ ab, int64_t lda, int64_t m, zval* __restrict__ out) {
  const int64_t n = 2 * m, total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % n, c = idx / n;
    const int64_t rr = r % m, cc = c % m;
    const bool low = r >= m, right = c >= m;
    // block (low,right): (0,0)=A (0,1)=B (1,0)=conj B (1,1)=conj A
    const bool use_b = low != right;
    zval v = ab[(use_b ? m + cc : cc) * lda + rr];
    if (low) v.im = -v.im;
    out[idx] = v;
  }
}

}  // namespace bse

namespace bse {

// a (k x k, ld = k) <- identity
__global__ void set_identity_kernel(zval* a, int k) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x)
    a[idx] = zval{(idx % k) == (idx / k) ? 1.0 : 0.0, 0.0};
}

__global__ void sqrt_kernel(const double* __restrict__ in, double* __restrict__ out, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = sqrt(in[i]);
}

// a_ii += s
__global__ void add_diag_kernel(zval* a, int k, double s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) a[(int64_t)i * k + i].re += s;
}

// per-column sum of |x|^2 over rows (one CTA per column), output squared norms
__global__ void frob2_kernel(const zval* __restrict__ x, int64_t ldx, int64_t n, double* __restrict__ out) {
  __shared__ double sh[32];
  const zval* col = x + (int64_t)blockIdx.x * ldx;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const zval v = col[i];
    s += v.re * v.re + v.im * v.im;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// |diag(R)| of a k x k upper factor into out
__global__ void absdiag_kernel(const zval* __restrict__ r, int k, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) {
    const zval v = r[(int64_t)i * k + i];
    out[i] = hypot(v.re, v.im);
  }
}

// g (k x k) <- diag(1/d) * g ; d real (rayleigh_ritz.py:168)
__global__ void rowscale_inv_kernel(zval* g, int k, const double* __restrict__ d) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = int(idx % k);
    zval v = g[idx];
    v.re /= d[i];
    v.im /= d[i];
    g[idx] = v;
  }
}

// off-diagonal part of m (diag zeroed) into out
__global__ void offdiag_kernel(const zval* __restrict__ m, zval* __restrict__ out, int k) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x)
    out[idx] = ((idx % k) == (idx / k)) ? zval{0.0, 0.0} : m[idx];
}

// real parts of the diagonal, zero entries (|d| <= tol) replaced by 1
__global__ void diag_real_kernel(const zval* __restrict__ m, int k, double tol, double* __restrict__ d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) {
    const double v = m[(int64_t)i * k + i].re;
    d[i] = fabs(v) <= tol ? 1.0 : v;
  }
}

}  // namespace bse

namespace bse {

// splitmix64 word at counter c (bsesolve/rng.py:37-42): exact integer math
__device__ __forceinline__ uint64_t sm64_word(uint64_t seed, uint64_t c) {
  uint64_t z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// complex normals start..start+count-1 (rng.py:63-75) with device libm
// (log/sincospi are within ~1 ulp of the host's; the words are bit-exact)
__global__ void complex_normals_kernel(zval* __restrict__ out, uint64_t seed, int64_t start, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t c = 2ull * (uint64_t)(start + i);
    const double u1 = ((double)(sm64_word(seed, c) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = ((double)(sm64_word(seed, c + 1) >> 11) + 1.0) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.141592653589793 * u2;
    double s, co;
    sincos(ang, &s, &co);
    out[i] = zval{r * co, r * s};
  }
}

// out (cols x rows, column-major) = transpose of the rows x cols column-major normal matrix:
// out[c + r*cols] <- normal #(c*rows + r)  (coalesced writes, counter-based draws)
__global__ void complex_normals_t_kernel(zval* __restrict__ out, uint64_t seed, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = o % cols, r = o / cols;  // out is cols x rows: element (c, r)
    const uint64_t ctr = 2ull * (uint64_t)(c * rows + r);
    const double u1 = ((double)(sm64_word(seed, ctr) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = ((double)(sm64_word(seed, ctr + 1) >> 11) + 1.0) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double s, co;
    sincos(2.0 * 3.141592653589793 * u2, &s, &co);
    out[o] = zval{rad * co, rad * s};
  }
}

// a (m x m, ld) <- (a + op(a)) / 2 with op = transpose (conj = 0) or conjugate transpose (conj = 1)
__global__ void symmetrize_kernel(zval* a, int64_t ld, int64_t m, int conj) {
  const int64_t total = m * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    if (i > j) continue;
    const zval x = a[j * ld + i], y = a[i * ld + j];
    const double yi = conj ? -y.im : y.im;
    const zval s{(x.re + y.re) / 2.0, (x.im + yi) / 2.0};
    a[j * ld + i] = s;
    a[i * ld + j] = zval{s.re, conj ? -s.im : s.im};
  }
}

// a <- scale * conj?(a) + shift * I  (m x m, ld)
__global__ void scale_shift_kernel(zval* a, int64_t ld, int64_t m, double scale, double shift, int conj) {
  const int64_t total = m * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    zval v = a[j * ld + i];
    v.re *= scale;
    v.im *= conj ? -scale : scale;
    if (i == j) v.re += shift;
    a[j * ld + i] = v;
  }
}

}  // namespace bse

namespace bse {

// Residual partials from the RR intermediate: with T = S H Q and V = Q w / d,
// H V = S T w / d, so  out[j] = sum_i | sgn_i u_ij uscale_j - lam_j v_ij |^2  with u = T w,
// sgn_i = -1 on rows >= half.  One CTA per column, fixed-order block reduction.
__global__ void resid_from_rr_kernel(const zval* __restrict__ u, int64_t ldu, const zval* __restrict__ v, int64_t ldv,
                                     int64_t rows, int64_t half, const double* __restrict__ uscale,
                                     const double* __restrict__ lam, double* __restrict__ out) {
  __shared__ double sh[32];
  const int64_t j = blockIdx.x;
  const zval* uc = u + j * ldu;
  const zval* vc = v + j * ldv;
  const double sc = uscale[j], l = lam[j];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const zval a = uc[i], b = vc[i];
    const double g = (i >= half) ? -sc : sc;
    const double rr = g * a.re - l * b.re, ri = g * a.im - l * b.im;
    s += rr * rr + ri * ri;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[j] = s;
}

__global__ void recip_kernel(const double* __restrict__ in, double* __restrict__ out, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = 1.0 / in[i];
}

}  // namespace bse

namespace bse {

// sd[i, j] = (re + im, re - im) of an m x cols column-major block (3M operand sums, built once)
__global__ void sum_planes_kernel(const zval* __restrict__ a, int64_t lda, int64_t m, int64_t cols,
                                  zval* __restrict__ sd) {
  const int64_t total = m * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    const zval v = a[j * lda + i];
    sd[j * lda + i] = zval{v.re + v.im, v.re - v.im};
  }
}

}  // namespace bse
