// Fused H-operator kernel: one complex FP64 GEMM that applies the BSE
// Hamiltonian H = [[A, B], [-conj(B), -conj(A)]] from its two stored blocks
// and finishes the result in the epilogue (Chebyshev three-term axpby,
// S-flip, or residual column norms), so no separate elementwise pass touches
// HBM.
//
// Reference semantics (paths under /root/reference/pkg/src/bsesolve/):
//   apply_h            hamiltonian.py:132-151   H x = [A x1 + B x2 ; -conj(A conj x2 + B conj x1)]
//   chebyshev_filter   chebyshev.py:68-74       y+ = (2s'/e)(H y - c y) - (s s') y-
//   build_hermitian_rq rayleigh_ritz.py:112      T = S H Q
//   residuals          rayleigh_ritz.py:188-189 ||H v - lam v||_2
//
// Formulation.  With P the current K-slab of A (part 0) or B (part 1):
//   U  += P    * Xa      (Xa = X1 for part 0, X2 for part 1)
//   L' += conj(P) * Xb   (Xb = X2 for part 0, X1 for part 1)
// and H x = [U ; -L'].  Both products share every P fragment, so the A/B
// stream is read once for the up and low halves.  Per 8x8 output block pair
// and k4 step: 8 DMMA (4M complex split), fragments via LDS.128.
#pragma once
#include "common.cuh"

namespace bse {

enum HopEpi : int { HOP_AXPBY = 0, HOP_RESID = 1 };

struct HopArgs {
  // P operand: part 0 (A tile) and part 1 (B tile), both mr x kc, column-major, leading dim lda
  const zval* pa;
  const zval* pb;
  int64_t lda;
  // 3M with precomputed operand sums (CM == 6): (Pr + Pi, Pr - Pi) planes of the same tiles
  const zval* sa;
  const zval* sb;
  int mr;  // output rows per half
  int kc;  // contraction length per part
  int skip_b;  // B == 0 (TDA / hermitian limit): contract over the A part only (4 n^2 k flops)
  // X operand rows for the contraction: x1 (rows of the "upper" half), x2 ("lower")
  const zval* x1;
  const zval* x2;
  int64_t ldx;
  int k;  // columns
  // epilogue operands (rows of the output)
  zval* y1;
  zval* y2;
  int64_t ldy;
  const zval* s1;  // shift operand (x at output rows); may be null when shift == 0
  const zval* s2;
  int64_t lds;
  const zval* p1;  // y_prev at output rows; may be null when beta == 0
  const zval* p2;
  int64_t ldp;
  double alpha, beta, shift, low_sign;
  // the shift term applies to output rows [shift_lo, shift_hi) only (the rows this tile's
  // input block shares with its output block in the 2D layout); per-column shifts when set
  int shift_lo, shift_hi;
  const double* shift_col;
  int group_rows;  // real-split kernel CTA raster (hop_rs.cuh); 0 = column tiles fastest
  // real-split split-K (hop_rs.cuh): ksplit > 1 CTAs share a tile's K range (gridDim.z) and write raw
  // partial sums to part_ws [z][h][col][row]; rs_splitk_epilogue_kernel sums and finishes them
  int ksplit;
  zval* part_ws;
  // fused group reduction (dist.py, 2D grid): npush > 0 -> the real-split output tile is stored to
  // npush peers' inbox slots (this rank's slot in each group member's symmetric buffer, NVLink
  // stores from the epilogue) instead of y1 / y2; y2's offset from y1 carries over to each target
  int npush;
  zval* push[4];
  // residual mode
  const double* lam;  // per column
  double* partial;    // [gridDim.y][k]
};

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_, int PS_ = 0>
struct HopCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_, PS = PS_;
  static constexpr int WARPS_M = BM / (8 * WM);
  static constexpr int WARPS_N = BN / (8 * WN);
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int LDP = BM + 2;  // == 2 (mod 8): conflict-free LDS.128 A fragments
  static constexpr int LDX = BK + 4;  // == 4 (mod 8): conflict-free LDS.128 B fragments
  static constexpr int P_ELEMS = BK * LDP;
  static constexpr int SD_ELEMS = PS ? BK * LDP : 0;  // (Pr+Pi, Pr-Pi) tile, same layout as P
  static constexpr int X_ELEMS = BN * LDX;
  static constexpr int STAGE_ELEMS = P_ELEMS + SD_ELEMS + 2 * X_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(zval);
  static_assert(BM % 8 == 0 && BK % 8 == 0 && BN % 8 == 0, "tile dims");
};

template <class C>
__device__ __forceinline__ void hop_load_stage(zval* st, const HopArgs& a, int kt, int nkt_part, int i0, int c0) {
  const int tid = threadIdx.x;
  const int part = kt >= nkt_part;
  const int j0 = (kt - part * nkt_part) * C::BK;
  const zval* P = part ? a.pb : a.pa;
  const zval* SD = part ? a.sb : a.sa;
  const zval* XA = part ? a.x2 : a.x1;
  const zval* XB = part ? a.x1 : a.x2;
  zval* Ps = st;
  zval* SDs = st + C::P_ELEMS;
  zval* Xas = SDs + C::SD_ELEMS;
  zval* Xbs = Xas + C::X_ELEMS;
#pragma unroll
  for (int r = 0; r < (C::BK * C::BM + C::THREADS - 1) / C::THREADS; ++r) {
    const int id = tid + r * C::THREADS;
    if ((C::BK * C::BM) % C::THREADS != 0 && id >= C::BK * C::BM) break;
    const int ii = id % C::BM, jj = id / C::BM;
    const int gi = i0 + ii, gj = j0 + jj;
    const bool ok = (gi < a.mr) && (gj < a.kc);
    const zval* src = ok ? P + (int64_t)gj * a.lda + gi : P;
    cp_async16(Ps + jj * C::LDP + ii, src, ok);
    if constexpr (C::PS == 1) cp_async16(SDs + jj * C::LDP + ii, ok ? SD + (int64_t)gj * a.lda + gi : SD, ok);
  }
#pragma unroll
  for (int r = 0; r < (2 * C::BN * C::BK + C::THREADS - 1) / C::THREADS; ++r) {
    const int id = tid + r * C::THREADS;
    if ((2 * C::BN * C::BK) % C::THREADS != 0 && id >= 2 * C::BN * C::BK) break;
    const int kk = id % C::BK;
    const int cc = (id / C::BK) % C::BN;
    const int which = id / (C::BK * C::BN);
    const int gj = j0 + kk, gc = c0 + cc;
    const bool ok = (gj < a.kc) && (gc < a.k);
    const zval* X = which ? XB : XA;
    const zval* src = ok ? X + (int64_t)gc * a.ldx + gj : X;
    cp_async16((which ? Xbs : Xas) + cc * C::LDX + kk, src, ok);
  }
}

// Per (i, j, h) accumulator values -> U = P Xa and L' = conj(P) Xb.
//  4M: acc = {Ur, Ui, L'r, L'i}.
//  3M: acc = {T1 = Pr Xar, T2 = Pi Xai, T3 = (Pr+Pi)(Xar+Xai), S1 = Pr Xbr, S2 = Pi Xbi, S3 = (Pr-Pi)(Xbr+Xbi)}
//      Ur = T1 - T2, Ui = T3 - T1 - T2, L'r = S1 + S2, L'i = S3 - S1 + S2.
template <int CM>
struct Acc {
  static constexpr int N = (CM == 3 || CM == 6) ? 6 : 4;
};

template <int CM, int WM, int WN>
__device__ __forceinline__ void acc_values(const double (&acc)[Acc<CM>::N][WM][WN][2], int i, int j, int h, double& ur,
                                           double& ui, double& lr, double& li) {
  if constexpr (CM == 3 || CM == 6) {
    const double t1 = acc[0][i][j][h], t2 = acc[1][i][j][h], t3 = acc[2][i][j][h];
    const double s1 = acc[3][i][j][h], s2 = acc[4][i][j][h], s3 = acc[5][i][j][h];
    ur = t1 - t2;
    ui = t3 - t1 - t2;
    lr = s1 + s2;
    li = s3 - s1 + s2;
  } else {
    ur = acc[0][i][j][h];
    ui = acc[1][i][j][h];
    lr = acc[2][i][j][h];
    li = acc[3][i][j][h];
  }
}

// Chebyshev / plain epilogue of one CTA tile: y = alpha (H x - shift x) - beta y_prev, lower half
// times low_sign, optional Re + Im planes of the output (shared by hop_kernel and hop3m_mb_kernel)
template <class C, int CM>
__device__ __forceinline__ void hop_epilogue_axpby(const double (&acc)[Acc<CM>::N][C::WM][C::WN][2], const HopArgs& a,
                                                   int i0, int c0, int wm, int wn, int g, int t) {
#pragma unroll
  for (int i = 0; i < C::WM; ++i) {
    const int row = i0 + wm * (8 * C::WM) + i * 8 + g;
    if (row >= a.mr) continue;
#pragma unroll
    for (int j = 0; j < C::WN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c0 + wn * (8 * C::WN) + j * 8 + 2 * t + h;
        if (col >= a.k) continue;
        // H x rows: up = U, low = -L'
        double hu_r, hu_i, hl_r, hl_i;
        acc_values<CM, C::WM, C::WN>(acc, i, j, h, hu_r, hu_i, hl_r, hl_i);
        hl_r = -hl_r;
        hl_i = -hl_i;
        if ((a.shift != 0.0 || a.shift_col) && row >= a.shift_lo && row < a.shift_hi) {
          const double sh = a.shift_col ? a.shift_col[col] : a.shift;
          const zval s1 = a.s1[(int64_t)col * a.lds + row];
          const zval s2 = a.s2[(int64_t)col * a.lds + row];
          hu_r = hu_r - sh * s1.re;
          hu_i = hu_i - sh * s1.im;
          hl_r = hl_r - sh * s2.re;
          hl_i = hl_i - sh * s2.im;
        }
        zval o1{a.alpha * hu_r, a.alpha * hu_i}, o2{a.alpha * hl_r, a.alpha * hl_i};
        if (a.beta != 0.0) {
          const zval q1 = a.p1[(int64_t)col * a.ldp + row];
          const zval q2 = a.p2[(int64_t)col * a.ldp + row];
          o1.re = o1.re - a.beta * q1.re;
          o1.im = o1.im - a.beta * q1.im;
          o2.re = o2.re - a.beta * q2.re;
          o2.im = o2.im - a.beta * q2.im;
        }
        o2.re *= a.low_sign;
        o2.im *= a.low_sign;
        a.y1[(int64_t)col * a.ldy + row] = o1;
        a.y2[(int64_t)col * a.ldy + row] = o2;
      }
    }
  }
}

template <class C, int EPI, int CM = 4>
__global__ void __launch_bounds__(C::THREADS, C::MINB) hop_kernel(const HopArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zval* smem = reinterpret_cast<zval*>(smem_raw);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int c0 = blockIdx.x * C::BN;  // column tile fastest: CTAs sharing an A/B strip run together
  const int i0 = blockIdx.y * C::BM;

  const int nkt_part = (a.kc + C::BK - 1) / C::BK;
  const int nkt = a.skip_b ? nkt_part : 2 * nkt_part;

  double acc[Acc<CM>::N][C::WM][C::WN][2];
#pragma unroll
  for (int q = 0; q < Acc<CM>::N; ++q)
#pragma unroll
    for (int i = 0; i < C::WM; ++i)
#pragma unroll
      for (int j = 0; j < C::WN; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;

  // prologue
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nkt) hop_load_stage<C>(smem + s * C::STAGE_ELEMS, a, s, nkt_part, i0, c0);
    cp_async_commit();
  }

  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + C::STAGES - 1;
      if (nxt < nkt) hop_load_stage<C>(smem + (nxt % C::STAGES) * C::STAGE_ELEMS, a, nxt, nkt_part, i0, c0);
      cp_async_commit();
    }
    const zval* Ps = smem + (kt % C::STAGES) * C::STAGE_ELEMS;
    const zval* SDs = Ps + C::P_ELEMS;
    const zval* Xas = SDs + C::SD_ELEMS;
    const zval* Xbs = Xas + C::X_ELEMS;
#pragma unroll
    for (int ks = 0; ks < C::BK / 4; ++ks) {
      zval pf[C::WM], xa[C::WN], xb[C::WN];
#pragma unroll
      for (int i = 0; i < C::WM; ++i) pf[i] = lds128(Ps + (ks * 4 + t) * C::LDP + wm * (8 * C::WM) + i * 8 + g);
#pragma unroll
      for (int j = 0; j < C::WN; ++j) {
        const int col = wn * (8 * C::WN) + j * 8 + g;
        xa[j] = lds128(Xas + col * C::LDX + ks * 4 + t);
        xb[j] = lds128(Xbs + col * C::LDX + ks * 4 + t);
      }
      if constexpr (CM == 6) {
        // 3M with the P-side sums read from shared memory
        zval sd[C::WM];
#pragma unroll
        for (int i = 0; i < C::WM; ++i) sd[i] = lds128(SDs + (ks * 4 + t) * C::LDP + wm * (8 * C::WM) + i * 8 + g);
        double xas[C::WN], xbs[C::WN];
#pragma unroll
        for (int j = 0; j < C::WN; ++j) {
          xas[j] = xa[j].re + xa[j].im;
          xbs[j] = xb[j].re + xb[j].im;
        }
#pragma unroll
        for (int i = 0; i < C::WM; ++i) {
#pragma unroll
          for (int j = 0; j < C::WN; ++j) {
            dmma(acc[0][i][j], pf[i].re, xa[j].re);
            dmma(acc[1][i][j], pf[i].im, xa[j].im);
            dmma(acc[2][i][j], sd[i].re, xas[j]);
            dmma(acc[3][i][j], pf[i].re, xb[j].re);
            dmma(acc[4][i][j], pf[i].im, xb[j].im);
            dmma(acc[5][i][j], sd[i].im, xbs[j]);
          }
        }
      } else if constexpr (CM == 3) {
        double xas[C::WN], xbs[C::WN];
#pragma unroll
        for (int j = 0; j < C::WN; ++j) {
          xas[j] = xa[j].re + xa[j].im;
          xbs[j] = xb[j].re + xb[j].im;
        }
#pragma unroll
        for (int i = 0; i < C::WM; ++i) {
          const double pr = pf[i].re, pi = pf[i].im;
          const double ps = pf[i].re + pf[i].im;
          const double pd = pf[i].re - pf[i].im;
#pragma unroll
          for (int j = 0; j < C::WN; ++j) {
            dmma(acc[0][i][j], pr, xa[j].re);
            dmma(acc[1][i][j], pi, xa[j].im);
            dmma(acc[2][i][j], ps, xas[j]);
            dmma(acc[3][i][j], pr, xb[j].re);
            dmma(acc[4][i][j], pi, xb[j].im);
            dmma(acc[5][i][j], pd, xbs[j]);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < C::WM; ++i) {
          const double pr = pf[i].re, pi = pf[i].im, npi = -pf[i].im;
#pragma unroll
          for (int j = 0; j < C::WN; ++j) {
            dmma(acc[0][i][j], pr, xa[j].re);
            dmma(acc[0][i][j], npi, xa[j].im);
            dmma(acc[1][i][j], pr, xa[j].im);
            dmma(acc[1][i][j], pi, xa[j].re);
            dmma(acc[2][i][j], pr, xb[j].re);
            dmma(acc[2][i][j], pi, xb[j].im);
            dmma(acc[3][i][j], pr, xb[j].im);
            dmma(acc[3][i][j], npi, xb[j].re);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  // ---------------------------------------------------------------- epilogue
  if constexpr (EPI == HOP_AXPBY) {
    hop_epilogue_axpby<C, CM>(acc, a, i0, c0, wm, wn, g, t);
  } else {
    // residual column norms: sum over this CTA's rows of |Hv - lam v|^2 (both halves)
    __shared__ double red[C::WARPS_M][C::BN];
    double rsum[C::WN][2];
#pragma unroll
    for (int j = 0; j < C::WN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = c0 + wn * (8 * C::WN) + j * 8 + 2 * t + h;
        double s = 0.0;
        if (col < a.k) {
          const double lam = a.lam[col];
#pragma unroll
          for (int i = 0; i < C::WM; ++i) {
            const int row = i0 + wm * (8 * C::WM) + i * 8 + g;
            if (row < a.mr) {
              const zval v1 = a.s1[(int64_t)col * a.lds + row];
              const zval v2 = a.s2[(int64_t)col * a.lds + row];
              double vur, vui, vlr, vli;
              acc_values<CM, C::WM, C::WN>(acc, i, j, h, vur, vui, vlr, vli);
              const double r1 = vur - lam * v1.re, r2 = vui - lam * v1.im;
              const double r3 = -vlr - lam * v2.re, r4 = -vli - lam * v2.im;
              s += r1 * r1 + r2 * r2 + r3 * r3 + r4 * r4;
            }
          }
        }
        // reduce across g (lane bits 2..4), fixed order
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        rsum[j][h] = s;
      }
    }
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < C::WN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) red[wm][wn * (8 * C::WN) + j * 8 + 2 * t + h] = rsum[j][h];
    }
    __syncthreads();
    for (int cc = threadIdx.x; cc < C::BN; cc += C::THREADS) {
      const int col = c0 + cc;
      if (col < a.k) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < C::WARPS_M; ++w) s += red[w][cc];
        a.partial[(int64_t)blockIdx.y * a.k + col] = s;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// k = 1 (Lanczos matvecs): the same operator as an HBM-bound split-K GEMV.  Thread = output
// row (coalesced column-major reads of the A and B tiles, x broadcast), per-split partials,
// fixed-order reduction.  Per launch: 32 mr kc bytes of A|B read once.
constexpr int GV_THREADS = 256;

__global__ void __launch_bounds__(GV_THREADS) gemv_partial_kernel(const zval* __restrict__ pa, const zval* __restrict__ pb,
                                                                  int64_t lda, int mr, int kc, const zval* __restrict__ x1,
                                                                  const zval* __restrict__ x2, int kchunk,
                                                                  zval* __restrict__ part, int skip_b) {
  const int i = blockIdx.x * GV_THREADS + threadIdx.x;
  const int j0 = blockIdx.y * kchunk, j1 = min(kc, j0 + kchunk);
  if (i >= mr) return;
  double ur = 0.0, ui = 0.0, lr = 0.0, li = 0.0;
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {
    const zval a = pa[(int64_t)j * lda + i];
    const zval b = skip_b ? zval{0.0, 0.0} : pb[(int64_t)j * lda + i];
    const zval p = x1[j], q = x2[j];
    ur += a.re * p.re - a.im * p.im + b.re * q.re - b.im * q.im;  // U  += a p + b q
    ui += a.re * p.im + a.im * p.re + b.re * q.im + b.im * q.re;
    lr += a.re * q.re + a.im * q.im + b.re * p.re + b.im * p.im;  // L' += conj(a) q + conj(b) p
    li += a.re * q.im - a.im * q.re + b.re * p.im - b.im * p.re;
  }
  zval* out = part + (int64_t)blockIdx.y * 2 * mr;
  out[i] = zval{ur, ui};
  out[mr + i] = zval{lr, li};
}

__global__ void gemv_reduce_kernel(const zval* __restrict__ part, int nsplit, int mr, zval* __restrict__ y1,
                                   zval* __restrict__ y2, double alpha, double low_sign) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 2 * mr) return;
  double sr = 0.0, si = 0.0;
  for (int z = 0; z < nsplit; ++z) {
    const zval v = part[(int64_t)z * 2 * mr + r];
    sr += v.re;
    si += v.im;
  }
  if (r < mr)
    y1[r] = zval{alpha * sr, alpha * si};
  else
    y2[r - mr] = zval{-low_sign * alpha * sr, -low_sign * alpha * si};  // low half of H x is -L'
}

}  // namespace bse
