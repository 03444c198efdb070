// Real-split ("RS") H operator: the filter product in the basis that diagonalises the
// pseudo-hermitian structure, 8 m^2 k real MACs per application instead of 12 m^2 k (3M) or
// 16 m^2 k (4M).
//
// With A = Ar + i Ai (hermitian) and B = Br + i Bi (symmetric), a state X = [X1; X2] is kept as
//   x = X1 + X2,   y = X1 - X2                                   (rs_fold_kernel)
// and H = [[A, B], [-conj B, -conj A]] (hamiltonian.py:132-151) acts on (x, y) as
//   x' = i Z x + V y,   y' = U x + i W y
// with the four REAL m x m planes
//   Z = Ai + Bi,  V = Ar - Br,  U = Ar + Br,  W = Ai - Bi        (rs_planes_kernel)
// (expand H X and collect the real and imaginary parts of X1' +- X2': the conjugations pair up so
// every plane multiplies a whole complex column).  A real plane times a complex column is 2 real
// products, so one application is 2 halves x 2 planes x 2 = 8 m^2 k DMMA MACs = 4 n^2 k flops,
// 2/3 of the 3M kernel's 6 n^2 k.  The filter's scalars (c, alpha, beta) are real, so the whole
// three-term recurrence (chebyshev.py:68-74) runs in the (x, y) basis and the block is unfolded
// once at the end (X1 = (x + y) / 2, X2 = (x - y) / 2; the factors of 2 are exact).
//
// Planes: one m x 4m real column-major array, plane q in columns [q m, (q + 1) m):
//   q = 0: Z, 1: V (output half x'), 2: U, 3: W (output half y').
// Output half h contracts plane 2h against x (part 0) and plane 2h + 1 against y (part 1); the
// pair (h, part) with h == part multiplies by i, done by rotating the B fragments in registers.
//
// Transposed-tile product (the 2D grid's row -> col step): the block
// transposes A[C_J, R_I] = A[R_I, C_J]^H, B[C_J, R_I] = B[R_I, C_J]^T have planes
//   Z' = -W^T,  V' = V^T,  U' = U^T,  W' = -Z^T
// (Ar, Br symmetric, Ai antisymmetric, Bi symmetric), so the same four planes serve both
// directions: TRANS reads them through a K-major TMA box (pitch BK + 4 doubles, == 4 mod 16:
// conflict-free LDS.64 again) and multiplies by -i where the forward product multiplies by i.
// A grid GPU therefore stores ONE tile's planes (32 m^2 / (p q) bytes) and nothing else.
//
// Feed: the TMA / producer-warp / mbarrier ring of hop3m_tma_kernel (hop_mb.cuh).  The real plane
// tile lands with pitch BM + 4 doubles (== 4 mod 16: the 16 lanes of each half warp read 16
// distinct 8-byte slots, conflict-free LDS.64), the complex X tile with pitch BK + 4 (LDS.128).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "hop_mb.cuh"
#include "tc_common.cuh"

namespace bse {

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_>
struct RsCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int WARPS_M = BM / (8 * WM);
  static constexpr int WARPS_N = BN / (8 * WN);
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;  // consumer threads (+ one producer warp)
  static constexpr int LDP = BM + 4;                      // doubles
  static constexpr int LDX = BK + 4;                      // complex
  static constexpr int LDK = BK + 4;                      // doubles (transposed plane tile)
  static constexpr int X_BYTES = BN * LDX * 16;
  template <bool TRANS>
  __host__ __device__ static constexpr int p_bytes() { return TRANS ? BM * LDK * 8 : BK * LDP * 8; }
  template <bool TRANS>
  __host__ __device__ static constexpr int stage_bytes() { return p_bytes<TRANS>() + X_BYTES; }
  template <bool TRANS>
  __host__ __device__ static constexpr size_t smem() { return size_t(STAGES) * stage_bytes<TRANS>() + 128; }
  static constexpr int P_BYTES = p_bytes<false>();
  static constexpr int STAGE_BYTES = stage_bytes<false>();
  static constexpr size_t SMEM = smem<false>();
  static_assert(BM % 16 == 0 && BN % 8 == 0 && BK % 4 == 0, "RS tile dims");
  static_assert(p_bytes<false>() % 128 == 0 && p_bytes<true>() % 128 == 0 && X_BYTES % 128 == 0,
                "TMA destinations must stay 128-byte aligned");
  static_assert(LDP <= 256 && LDK <= 256 && 2 * LDX <= 256 && BN <= 256 && BK <= 256, "TMA box dimensions");
};

// Arguments: HopArgs (hop.cuh) with x1 / x2 = the x / y parts of the folded input (kc rows each),
// y1 / y2 = the x' / y' halves of the output (mr rows each), s1 / s2 and p1 / p2 likewise; the
// epilogue is hop_epilogue_axpby's with low_sign == 1 (pa, pb, sa, sb, skip_b unused).
struct RsMaps {
  CUtensorMap g[4];  // planes Z, V, U, W of the tile: mr x kc doubles each, leading dim ldg
  CUtensorMap x[2];  // x and y parts of the input: (2 kc doubles) x k, leading dim 2 ldx
};

// One k4 slice of a warp's operands: plane fragment (A of DMMA.8x8x4) and the real / imaginary
// parts of the input fragment (B), the latter already multiplied by rot i (rot = 0, +1, -1; the
// sign flips are exact, so the products are those of the unrotated form bit for bit).
template <class C>
struct RsFrag {
  double pf[C::WM];
  double br[C::WN], bi[C::WN];
};

// ROT: 0 -> x, +1 -> i x, -1 -> -i x; TRANS: the plane tile is K-major (see the header)
template <int ROT, bool TRANS, class C>
__device__ __forceinline__ void rs_load_frag_t(RsFrag<C>& f, const double* Ps, const zval* Xs, int ks, int wm, int wn,
                                               int g, int t) {
#pragma unroll
  for (int i = 0; i < C::WM; ++i) {
    const int r = wm * (8 * C::WM) + i * 8 + g;
    f.pf[i] = TRANS ? Ps[r * C::LDK + ks * 4 + t] : Ps[(ks * 4 + t) * C::LDP + r];
  }
#pragma unroll
  for (int j = 0; j < C::WN; ++j) {
    const zval xv = lds128(Xs + (wn * (8 * C::WN) + j * 8 + g) * C::LDX + ks * 4 + t);
    if constexpr (ROT > 0) {
      f.br[j] = -xv.im;
      f.bi[j] = xv.re;
    } else if constexpr (ROT < 0) {
      f.br[j] = xv.im;
      f.bi[j] = -xv.re;
    } else {
      f.br[j] = xv.re;
      f.bi[j] = xv.im;
    }
  }
}

// PARTIAL: only the first nv 8-column fragments of the warp hold columns < k (the last column
// tile of a block whose width is not a multiple of BN); the others are skipped (warp-uniform)
template <class C, bool PARTIAL = false>
__device__ __forceinline__ void rs_mma(double (&acc)[2][C::WM][C::WN][2], const RsFrag<C>& f, int nv = C::WN) {
#pragma unroll
  for (int i = 0; i < C::WM; ++i)
#pragma unroll
    for (int j = 0; j < C::WN; ++j) {
      if (PARTIAL && j >= nv) continue;
      dmma(acc[0][i][j], f.pf[i], f.br[j]);
      dmma(acc[1][i][j], f.pf[i], f.bi[j]);
    }
}

// output store of half h at element idx = col * ldy + row: local y, or every push target
__device__ __forceinline__ void rs_store(const HopArgs& a, int h, int64_t idx, const zval& out) {
  if (a.npush > 0) {
    const int64_t off = h ? (a.y2 - a.y1) : 0;
#pragma unroll 1
    for (int r = 0; r < a.npush; ++r) a.push[r][off + idx] = out;
  } else {
    (h ? a.y2 : a.y1)[idx] = out;
  }
}

// grid: x = column tiles (fastest: CTAs sharing a plane strip run together), y = 2 * row tiles
// plane read by output half h for input part (0: x, 1: y): forward Z V | U W, transposed W V | U Z
template <bool TRANS>
__device__ __forceinline__ int rs_plane(int h, int part) {
  return TRANS ? (h ? (part ? 0 : 2) : (part ? 1 : 3)) : 2 * h + part;
}

// GENERIC: fragment loads through a generic pointer (LD) instead of shared-space LDS -- measured
// faster for the 128 x 32 tile, slower for the 64 x 32 one (profiles/r02/rs_consumer_variants_*.txt;
// a slice-ahead software-pipelined consumer measured 3-9% slower than both and was dropped)
// PUSH: the fused group reduction's instantiation (stores through rs_store to the push targets);
// the default one keeps the plain local store, so its code is unchanged by the feature
template <class C, bool TRANS = false, bool GENERIC = false, bool PUSH = false>
__global__ void __launch_bounds__(C::THREADS + 32, C::MINB) hop_rs_tma_kernel(const HopArgs a,
                                                                              const __grid_constant__ RsMaps maps) {
  constexpr int P_BYTES = C::template p_bytes<TRANS>();
  constexpr int STAGE_BYTES = C::template stage_bytes<TRANS>();
  constexpr int NWARPS = C::THREADS / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base =
      GENERIC ? reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127))
             : smem_raw + (((128u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int nbm = (a.mr + C::BM - 1) / C::BM;
  // CTA raster: by default column tiles run fastest (the CTAs of one plane strip run together); with
  // GROUP_ROWS > 0 the launch order walks GROUP_ROWS row tiles per column tile first, so a wave spans
  // fewer column tiles of X (X is re-streamed once per wave: the bulk of the DRAM traffic)
  int row_tile = blockIdx.y, col_tile = blockIdx.x;
  if (a.group_rows > 0) {
    const int ncol = gridDim.x, nrow = gridDim.y;
    const int pid = blockIdx.y * ncol + blockIdx.x;
    const int per_group = a.group_rows * ncol;
    const int grp = pid / per_group, first = grp * a.group_rows;
    const int rows_here = min(a.group_rows, nrow - first);
    row_tile = first + (pid % per_group) % rows_here;
    col_tile = (pid % per_group) / rows_here;
  }
  const int h = row_tile >= nbm;  // output half: 0 -> x', 1 -> y'
  const int i0 = (row_tile - h * nbm) * C::BM;
  const int c0 = col_tile * C::BN;
  const int nkt_part = (a.kc + C::BK - 1) / C::BK;
  // this CTA's K stages [kt0, kt1) of the 2 nkt_part (all of them unless split-K)
  const int nsplit = a.ksplit > 1 ? a.ksplit : 1;
  const int per_split = (2 * nkt_part + nsplit - 1) / nsplit;
  const int kt0 = min(2 * nkt_part, (int)blockIdx.z * per_split);
  const int nkt = min(2 * nkt_part, kt0 + per_split) - kt0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init_cta(&full[s], 1);
      mbar_init_cta(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    tc::prefetch_tmap(&maps.g[rs_plane<TRANS>(h, 0)]);
    tc::prefetch_tmap(&maps.g[rs_plane<TRANS>(h, 1)]);
    tc::prefetch_tmap(&maps.x[0]);
    tc::prefetch_tmap(&maps.x[1]);
  }
  __syncthreads();

  if (warp == NWARPS) {
    if (lane == 0) {
      for (int lkt = 0; lkt < nkt; ++lkt) {
        const int b = lkt % C::STAGES;
        if (lkt >= C::STAGES) mbar_wait_cta(&empty[b], ((lkt - C::STAGES) / C::STAGES) & 1);
        const int gkt = kt0 + lkt;
        const int part = gkt >= nkt_part;
        const int j0 = (gkt - part * nkt_part) * C::BK;
        unsigned char* st = base + b * STAGE_BYTES;
        tc::mbar_arrive_expect_tx(&full[b], STAGE_BYTES);
        if (TRANS)
          tc::tma_load_2d(st, &maps.g[rs_plane<TRANS>(h, part)], &full[b], j0, i0);
        else
          tc::tma_load_2d(st, &maps.g[rs_plane<TRANS>(h, part)], &full[b], i0, j0);
        tc::tma_load_2d(st + P_BYTES, &maps.x[part], &full[b], 2 * j0, c0);
      }
    }
    return;
  }

  double acc[2][C::WM][C::WN][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int i = 0; i < C::WM; ++i)
#pragma unroll
      for (int j = 0; j < C::WN; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;

  constexpr int KS = C::BK / 4;
  auto stage_p = [&](int s) { return reinterpret_cast<const double*>(base + s * STAGE_BYTES); };
  auto stage_x = [&](int s) { return reinterpret_cast<const zval*>(base + s * STAGE_BYTES + P_BYTES); };
  // 8-column fragments of this warp that hold columns < k: all of them except in the last column
  // tile of a ragged block, where the rest are skipped (same bits for the valid columns)
  const int nv = min(C::WN, max(0, (a.k - c0 - wn * 8 * C::WN + 7) / 8));
  auto consume = [&](auto partial) {
    constexpr bool PARTIAL = decltype(partial)::value;
#pragma unroll 1
    for (int kt = 0; kt < nkt; ++kt) {
      const int s = kt % C::STAGES;
      mbar_wait_cta(&full[s], (kt / C::STAGES) & 1);
      const double* Ps = stage_p(s);
      const zval* Xs = stage_x(s);
      RsFrag<C> f;
      if ((kt0 + kt >= nkt_part) == (h == 1)) {  // the i (forward) / -i (transposed) part of this half
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          rs_load_frag_t<TRANS ? -1 : 1, TRANS, C>(f, Ps, Xs, ks, wm, wn, g, t);
          rs_mma<C, PARTIAL>(acc, f, nv);
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          rs_load_frag_t<0, TRANS, C>(f, Ps, Xs, ks, wm, wn, g, t);
          rs_mma<C, PARTIAL>(acc, f, nv);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
    }
  };
  if (nv < C::WN)
    consume(std::true_type{});
  else
    consume(std::false_type{});

  if (nsplit > 1) {  // raw partial sums; rs_splitk_epilogue_kernel finishes the output
    zval* w = a.part_ws + ((int64_t)(blockIdx.z * 2 + h) * a.k) * a.mr;
#pragma unroll
    for (int i = 0; i < C::WM; ++i) {
      const int row = i0 + wm * (8 * C::WM) + i * 8 + g;
      if (row >= a.mr) continue;
#pragma unroll
      for (int j = 0; j < C::WN; ++j)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int col = c0 + wn * (8 * C::WN) + j * 8 + 2 * t + hh;
          if (col < a.k) w[(int64_t)col * a.mr + row] = zval{acc[0][i][j][hh], acc[1][i][j][hh]};
        }
    }
    return;
  }

  // epilogue: y_h = alpha (acc - shift s_h) - beta p_h on the output half h
  zval* yh = h ? a.y2 : a.y1;
  const zval* sh = h ? a.s2 : a.s1;
  const zval* ph = h ? a.p2 : a.p1;
#pragma unroll
  for (int i = 0; i < C::WM; ++i) {
    const int row = i0 + wm * (8 * C::WM) + i * 8 + g;
    if (row >= a.mr) continue;
    const bool shifted = (a.shift != 0.0 || a.shift_col) && row >= a.shift_lo && row < a.shift_hi;
#pragma unroll
    for (int j = 0; j < C::WN; ++j) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int col = c0 + wn * (8 * C::WN) + j * 8 + 2 * t + hh;
        if (col >= a.k) continue;
        double vr = acc[0][i][j][hh], vi = acc[1][i][j][hh];
        if (shifted) {
          const double sc = a.shift_col ? a.shift_col[col] : a.shift;
          const zval s = sh[(int64_t)col * a.lds + row];
          vr = vr - sc * s.re;
          vi = vi - sc * s.im;
        }
        zval out{a.alpha * vr, a.alpha * vi};
        if (a.beta != 0.0) {
          const zval p = ph[(int64_t)col * a.ldp + row];
          out.re = out.re - a.beta * p.re;
          out.im = out.im - a.beta * p.im;
        }
        if constexpr (PUSH)
          rs_store(a, h, (int64_t)col * a.ldy + row, out);
        else
          yh[(int64_t)col * a.ldy + row] = out;
      }
    }
  }
}

// split-K finish: y_h = alpha (sum_z part[z][h] - shift s_h) - beta p_h, the partials added in a
// fixed order (deterministic), the same epilogue arithmetic as hop_rs_tma_kernel's
__global__ void rs_splitk_epilogue_kernel(const HopArgs a) {
  const int64_t total = 2 * (int64_t)a.k * a.mr;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = int(idx % a.mr);
    const int64_t rest = idx / a.mr;
    const int col = int(rest % a.k), h = int(rest / a.k);
    double vr = 0.0, vi = 0.0;
    for (int z = 0; z < a.ksplit; ++z) {
      const zval v = a.part_ws[((int64_t)(z * 2 + h) * a.k + col) * a.mr + row];
      vr += v.re;
      vi += v.im;
    }
    if ((a.shift != 0.0 || a.shift_col) && row >= a.shift_lo && row < a.shift_hi) {
      const double sc = a.shift_col ? a.shift_col[col] : a.shift;
      const zval s = (h ? a.s2 : a.s1)[(int64_t)col * a.lds + row];
      vr = vr - sc * s.re;
      vi = vi - sc * s.im;
    }
    zval out{a.alpha * vr, a.alpha * vi};
    if (a.beta != 0.0) {
      const zval p = (h ? a.p2 : a.p1)[(int64_t)col * a.ldp + row];
      out.re = out.re - a.beta * p.re;
      out.im = out.im - a.beta * p.im;
    }
    rs_store(a, h, (int64_t)col * a.ldy + row, out);
  }
}

// y = sum_j inbox[j] over the nslot slots of a group's symmetric buffer, in slot order (the fused
// group reduction's second half: every member adds the same partials in the same order)
__global__ void group_sum_kernel(const zval* __restrict__ inbox, int64_t stride, int nslot, zval* __restrict__ y,
                                 int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    zval v = inbox[i];
    for (int j = 1; j < nslot; ++j) {
      const zval w = inbox[j * stride + i];
      v.re += w.re;
      v.im += w.im;
    }
    y[i] = v;
  }
}

// planes of a tile [A_t | B_t] (mr x 2kc complex, leading dim lda) -> mr x 4kc real (leading dim ldg)
__global__ void rs_planes_kernel(const zval* __restrict__ ab, int64_t lda, int64_t mr, int64_t kc, double* __restrict__ gp,
                                 int64_t ldg) {
  const int64_t total = mr * kc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % mr, j = idx / mr;
    const zval av = ab[j * lda + i];
    const zval bv = ab[(kc + j) * lda + i];
    gp[j * ldg + i] = av.im + bv.im;             // Z
    gp[(kc + j) * ldg + i] = av.re - bv.re;      // V
    gp[(2 * kc + j) * ldg + i] = av.re + bv.re;  // U
    gp[(3 * kc + j) * ldg + i] = av.im - bv.im;  // W
  }
}

// (X1, X2) -> (scale (X1 + X2), scale2 (X1 - X2)): fold with 1, 1; unfold with 1/2, 1/2 (S-flipped:
// 1/2, -1/2); src may equal dst (same leading dimension then)
__global__ void rs_fold_kernel(const zval* src, zval* dst, int64_t lds, int64_t ldd, int64_t m, int64_t k, double scale,
                               double scale2) {
  const int64_t total = m * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    const zval a = src[j * lds + i], b = src[j * lds + m + i];
    dst[j * ldd + i] = zval{scale * (a.re + b.re), scale * (a.im + b.im)};
    dst[j * ldd + m + i] = zval{scale2 * (a.re - b.re), scale2 * (a.im - b.im)};
  }
}

}  // namespace bse
