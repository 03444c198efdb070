// Complex FP64 GEMM on the DMMA pipe for the tall-skinny products of the
// orthonormalisation and Rayleigh-Ritz phases:
//   OPA_C :  C(MxN) = alpha * A^H B + beta * C    (A: K x M, B: K x N; Gram-type, K = n)
//   OPA_N :  C(MxN) = alpha * A   B + beta * C    (A: M x K, B: K x N; basis update Q*W)
// All operands column-major complex128.  Split-K (gridDim.z > 1) writes
// per-split partials that zgemm_splitk_reduce sums in a fixed order, so the
// result is deterministic run to run (no atomics).
//
// Reference call sites replaced (bsesolve/): ortho.py:116 (q^H q), :124
// (defect q^H q - I), :152 (basis^H v, basis @ .), rayleigh_ritz.py:113
// (Q^H T), :93 (Q2^H Q2), :135 (Q @ w).
#pragma once
#include "common.cuh"

namespace bse {

enum : int { OPA_N = 0, OPA_C = 1 };

struct GemmArgs {
  const zval* a;
  int64_t lda;
  const zval* b;
  int64_t ldb;
  zval* c;
  int64_t ldc;
  int M, N, K;
  double alpha, beta;
  zval* ws;  // split-K partials [z][N][M] (ld = M), used when gridDim.z > 1
  // structure: GEMM_UPPER -- only tiles touching the upper triangle are computed (a hermitian
  // result, M == N; the strictly lower part is left undefined for herm_upper_kernel to fill);
  // GEMM_B_UPPER -- B is upper triangular (K == N), so output column j needs K rows <= j only
  int tri;
};
enum : int { GEMM_UPPER = 1, GEMM_B_UPPER = 2 };

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int WARPS_M = BM / (8 * WM);
  static constexpr int WARPS_N = BN / (8 * WN);
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int LDN = BM + 2;  // OPA_N tile [k][m]
  static constexpr int LDK = BK + 4;  // OPA_C tile [m][k] and B tile [n][k]
  static constexpr int A_ELEMS_N = BK * LDN;
  static constexpr int A_ELEMS_C = BM * LDK;
  static constexpr int A_ELEMS = A_ELEMS_N > A_ELEMS_C ? A_ELEMS_N : A_ELEMS_C;
  static constexpr int B_ELEMS = BN * LDK;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(zval);
  static_assert((BK * BM) % THREADS == 0 && (BK * BN) % THREADS == 0, "loader mapping");
};

template <class C, int OPA>
__device__ __forceinline__ void gemm_load_stage(zval* st, const GemmArgs& g, int k0, int i0, int j0) {
  const int tid = threadIdx.x;
  zval* As = st;
  zval* Bs = st + C::A_ELEMS;
#pragma unroll
  for (int r = 0; r < (C::BK * C::BM) / C::THREADS; ++r) {
    const int id = tid + r * C::THREADS;
    if constexpr (OPA == OPA_N) {
      const int ii = id % C::BM, kk = id / C::BM;
      const bool ok = (i0 + ii < g.M) && (k0 + kk < g.K);
      const zval* src = ok ? g.a + (int64_t)(k0 + kk) * g.lda + i0 + ii : g.a;
      cp_async16(As + kk * C::LDN + ii, src, ok);
    } else {
      const int kk = id % C::BK, ii = id / C::BK;
      const bool ok = (i0 + ii < g.M) && (k0 + kk < g.K);
      const zval* src = ok ? g.a + (int64_t)(i0 + ii) * g.lda + k0 + kk : g.a;
      cp_async16(As + ii * C::LDK + kk, src, ok);
    }
  }
#pragma unroll
  for (int r = 0; r < (C::BK * C::BN) / C::THREADS; ++r) {
    const int id = tid + r * C::THREADS;
    const int kk = id % C::BK, jj = id / C::BK;
    const bool ok = (j0 + jj < g.N) && (k0 + kk < g.K);
    const zval* src = ok ? g.b + (int64_t)(j0 + jj) * g.ldb + k0 + kk : g.b;
    cp_async16(Bs + jj * C::LDK + kk, src, ok);
  }
}

template <class C, int OPA>
__global__ void __launch_bounds__(C::THREADS) zgemm_kernel(const GemmArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zval* smem = reinterpret_cast<zval*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int i0 = blockIdx.x * C::BM, j0 = blockIdx.y * C::BN;
  if ((g.tri & GEMM_UPPER) && i0 >= j0 + C::BN) return;  // tile strictly below the diagonal
  const int K = (g.tri & GEMM_B_UPPER) ? min(g.K, j0 + C::BN) : g.K;

  // split-K range
  const int nkt_all = (K + C::BK - 1) / C::BK;
  const int per = (nkt_all + gridDim.z - 1) / gridDim.z;
  const int kt_begin = blockIdx.z * per;
  const int kt_end = min(nkt_all, kt_begin + per);
  const int nkt = max(0, kt_end - kt_begin);

  double cr[C::WM][C::WN][2], ci[C::WM][C::WN][2];
#pragma unroll
  for (int i = 0; i < C::WM; ++i)
#pragma unroll
    for (int j = 0; j < C::WN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nkt) gemm_load_stage<C, OPA>(smem + s * C::STAGE_ELEMS, g, (kt_begin + s) * C::BK, i0, j0);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + C::STAGES - 1;
      if (nxt < nkt) gemm_load_stage<C, OPA>(smem + (nxt % C::STAGES) * C::STAGE_ELEMS, g, (kt_begin + nxt) * C::BK, i0, j0);
      cp_async_commit();
    }
    const zval* As = smem + (kt % C::STAGES) * C::STAGE_ELEMS;
    const zval* Bs = As + C::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < C::BK / 4; ++ks) {
      zval af[C::WM], bf[C::WN];
#pragma unroll
      for (int i = 0; i < C::WM; ++i) {
        const int mm = wm * (8 * C::WM) + i * 8 + gq;
        if constexpr (OPA == OPA_N)
          af[i] = lds128(As + (ks * 4 + t) * C::LDN + mm);
        else
          af[i] = lds128(As + mm * C::LDK + ks * 4 + t);
      }
#pragma unroll
      for (int j = 0; j < C::WN; ++j) bf[j] = lds128(Bs + (wn * (8 * C::WN) + j * 8 + gq) * C::LDK + ks * 4 + t);
#pragma unroll
      for (int i = 0; i < C::WM; ++i) {
        const double ar = af[i].re, ai = af[i].im, nai = -af[i].im;
#pragma unroll
        for (int j = 0; j < C::WN; ++j) {
          if constexpr (OPA == OPA_N) {
            dmma(cr[i][j], ar, bf[j].re);
            dmma(cr[i][j], nai, bf[j].im);
            dmma(ci[i][j], ar, bf[j].im);
            dmma(ci[i][j], ai, bf[j].re);
          } else {  // conj(A)
            dmma(cr[i][j], ar, bf[j].re);
            dmma(cr[i][j], ai, bf[j].im);
            dmma(ci[i][j], ar, bf[j].im);
            dmma(ci[i][j], nai, bf[j].re);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < C::WM; ++i) {
    const int row = i0 + wm * (8 * C::WM) + i * 8 + gq;
    if (row >= g.M) continue;
#pragma unroll
    for (int j = 0; j < C::WN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = j0 + wn * (8 * C::WN) + j * 8 + 2 * t + h;
        if (col >= g.N) continue;
        if (gridDim.z > 1) {
          g.ws[((int64_t)blockIdx.z * g.N + col) * g.M + row] = zval{cr[i][j][h], ci[i][j][h]};
        } else {
          zval o{g.alpha * cr[i][j][h], g.alpha * ci[i][j][h]};
          zval* dst = g.c + (int64_t)col * g.ldc + row;
          if (g.beta != 0.0) {
            const zval old = *dst;
            o.re += g.beta * old.re;
            o.im += g.beta * old.im;
          }
          *dst = o;
        }
      }
  }
}

// Fixed-order split-K sum: C = alpha * sum_z ws[z] + beta * C
__global__ void zgemm_splitk_reduce(const zval* __restrict__ ws, int splits, zval* c, int64_t ldc, int M, int N,
                                    double alpha, double beta, int tri) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = int(idx % M);
    const int64_t col = idx / M;
    if ((tri & GEMM_UPPER) && row > col) continue;  // partials of skipped tiles were never written
    double sr = 0.0, si = 0.0;
    for (int z = 0; z < splits; ++z) {
      const zval v = ws[(int64_t)z * total + idx];
      sr += v.re;
      si += v.im;
    }
    zval o{alpha * sr, alpha * si};
    zval* dst = c + col * ldc + row;
    if (beta != 0.0) {
      const zval old = *dst;
      o.re += beta * old.re;
      o.im += beta * old.im;
    }
    *dst = o;
  }
}

}  // namespace bse
