// 3M filter product fed by TMA through mbarrier rings (hop3m_tma_kernel), plus the mbarrier
// helpers the real-split kernel (hop_rs.cuh) shares.
//
// Every stage buffer has two mbarriers: full[s] (the producer's expect-tx arrival; the TMA bytes
// complete it) and empty[s] (one arrival per consumer warp once it has read the stage), so warps
// drift up to a stage apart instead of meeting at a CTA barrier.  The math is hop_kernel's
// CM == 6 3M split (hop.cuh): U = P Xa, L' = conj(P) Xb on the precomputed (Pr + Pi, Pr - Pi)
// planes; same epilogue.  (Round 1's cp.async-fed version of this pipeline is retired.)
#pragma once
#include <cuda.h>

#include "hop.cuh"
#include "tc_common.cuh"

namespace bse {

__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cta(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "MB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra MB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Stage layout: hop_kernel's padded tiles (LDP = BM + 2, LDX = BK + 4: conflict-free LDS.128).
// (An unpadded X tile with the K halves swapped on odd columns is conflict free too and saves a
// third of the X bytes; it measured no faster, profiles/r01/tune_3m_swizzle.txt.)
template <class C>
struct MbLayout {
  static constexpr int LDX = C::LDX;
  static constexpr int X_ELEMS = C::BN * LDX;
  static constexpr int STAGE_ELEMS = C::P_ELEMS + C::SD_ELEMS + 2 * X_ELEMS;
  static constexpr size_t SMEM = size_t(C::STAGES) * STAGE_ELEMS * sizeof(zval);
};

// the 3M DMMA work of one landed stage (identical arithmetic to hop_kernel CM == 6)
template <class C>
__device__ __forceinline__ void mb_stage_mma(double (&acc)[6][C::WM][C::WN][2], const zval* Ps, const zval* SDs,
                                             const zval* Xas, const zval* Xbs, int wm, int wn, int g, int t) {
  using L = MbLayout<C>;
#pragma unroll
  for (int ks = 0; ks < C::BK / 4; ++ks) {
    zval pf[C::WM], sdf[C::WM], xa[C::WN], xb[C::WN];
#pragma unroll
    for (int i = 0; i < C::WM; ++i) {
      pf[i] = lds128(Ps + (ks * 4 + t) * C::LDP + wm * (8 * C::WM) + i * 8 + g);
      if constexpr (C::PS == 1)
        sdf[i] = lds128(SDs + (ks * 4 + t) * C::LDP + wm * (8 * C::WM) + i * 8 + g);
      else  // no sum planes: the same FP64 adds as sum_planes_kernel, in registers
        sdf[i] = zval{pf[i].re + pf[i].im, pf[i].re - pf[i].im};
    }
#pragma unroll
    for (int j = 0; j < C::WN; ++j) {
      const int col = wn * (8 * C::WN) + j * 8 + g;
      xa[j] = lds128(Xas + col * L::LDX + ks * 4 + t);
      xb[j] = lds128(Xbs + col * L::LDX + ks * 4 + t);
    }
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
        dmma(acc[2][i][j], sdf[i].re, xas[j]);
        dmma(acc[3][i][j], pf[i].re, xb[j].re);
        dmma(acc[4][i][j], pf[i].im, xb[j].im);
        dmma(acc[5][i][j], sdf[i].im, xbs[j]);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// TMA-fed variant.  The padded shared layouts above (LDP = BM + 2, LDX = BK + 4) are what make the
// fragment LDS.128 conflict-free; a TMA box is written densely, so the boxes are made as wide as
// the padded rows: P / sum-plane boxes of (BM + 2) complex x BK rows land with pitch LDP, X boxes
// of (BK + 4) complex x BN columns land with pitch LDX (the extra rows / K values are neighbouring
// data or TMA's zero fill, never read).  A producer warp issues 4 bulk-tensor copies per stage
// against full[s] (arrive.expect_tx) instead of 8 cp.async per thread, and waits only on the
// empty barriers, so no consumer warp ever waits for another (with one consumer thread as the
// producer, warp 0 is throttled by the slowest warp: 7% slower, profiles/r01/tune_3m_tma.txt).
struct HopMaps {
  CUtensorMap p[2];   // [A | B] parts: (2 mr doubles) x kc, leading dim lda
  CUtensorMap sd[2];  // their (Pr + Pi, Pr - Pi) planes
  CUtensorMap x[2];   // x1, x2: (2 kc doubles) x k, leading dim ldx
};

template <class C>
struct TmaLayout {
  // PS == 1: P and its sum planes staged; PS == 0: P only, the sums formed in registers
  static_assert(C::PS == 0 || C::PS == 1, "TMA feed: 3M with or without P-side sum planes");
  static constexpr int P_BYTES = C::P_ELEMS * 16, X_BYTES = C::X_ELEMS * 16;
  static constexpr int NP = C::PS ? 2 : 1;  // P tiles per stage
  static constexpr int STAGE_BYTES = NP * P_BYTES + 2 * X_BYTES;
  static_assert(P_BYTES % 128 == 0 && X_BYTES % 128 == 0, "TMA destinations must stay 128-byte aligned");
  static_assert(2 * (C::BM + 2) <= 256 && 2 * (C::BK + 4) <= 256 && C::BN <= 256 && C::BK <= 256,
                "TMA box dimensions are limited to 256 elements");
  static constexpr size_t SMEM = size_t(C::STAGES) * STAGE_BYTES + 128;  // + alignment slack
};

// C::THREADS consumer threads + one producer warp (warp C::THREADS / 32)
template <class C>
__global__ void __launch_bounds__(C::THREADS + 32, C::MINB)
    hop3m_tma_kernel(const HopArgs a, const __grid_constant__ HopMaps maps) {
  using T = TmaLayout<C>;
  constexpr int CM = 6;
  constexpr int NWARPS = C::THREADS / 32;  // consumer warps
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base =
      smem_raw + (((128u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 127u)) & 127u));  // stays a shared-space pointer: LDS, not generic LD
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int c0 = blockIdx.x * C::BN;
  const int i0 = blockIdx.y * C::BM;
  const int nkt_part = (a.kc + C::BK - 1) / C::BK;
  const int nkt = a.skip_b ? nkt_part : 2 * nkt_part;
  const bool producer = threadIdx.x == C::THREADS;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init_cta(&full[s], 1);
      mbar_init_cta(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    for (int q = 0; q < 2; ++q) {
      tc::prefetch_tmap(&maps.p[q]);
      if constexpr (C::PS == 1) tc::prefetch_tmap(&maps.sd[q]);
      tc::prefetch_tmap(&maps.x[q]);
    }
  }
  __syncthreads();

  int lkt = 0;  // next stage to load (producer only)
  auto load_next = [&](int buf) {
    const int part = lkt >= nkt_part;
    const int j0 = (lkt - part * nkt_part) * C::BK;
    unsigned char* st = base + buf * T::STAGE_BYTES;
    tc::mbar_arrive_expect_tx(&full[buf], T::STAGE_BYTES);
    tc::tma_load_2d(st, &maps.p[part], &full[buf], 2 * i0, j0);
    if constexpr (C::PS == 1) tc::tma_load_2d(st + T::P_BYTES, &maps.sd[part], &full[buf], 2 * i0, j0);
    tc::tma_load_2d(st + T::NP * T::P_BYTES, &maps.x[part], &full[buf], 2 * j0, c0);                  // Xa
    tc::tma_load_2d(st + T::NP * T::P_BYTES + T::X_BYTES, &maps.x[1 - part], &full[buf], 2 * j0, c0);  // Xb
    ++lkt;
  };
  if (warp == NWARPS) {
    if (producer) {
      // run STAGES deep: the buffer of stage lkt last held stage lkt - STAGES
      for (int s = 0; s < C::STAGES && lkt < nkt; ++s) load_next(s);
      while (lkt < nkt) {
        const int b = lkt % C::STAGES;
        mbar_wait_cta(&empty[b], ((lkt - C::STAGES) / C::STAGES) & 1);
        load_next(b);
      }
    }
    return;
  }

  double acc[Acc<CM>::N][C::WM][C::WN][2];
#pragma unroll
  for (int q = 0; q < Acc<CM>::N; ++q)
#pragma unroll
    for (int i = 0; i < C::WM; ++i)
#pragma unroll
      for (int j = 0; j < C::WN; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;

#pragma unroll 1
  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % C::STAGES;
    mbar_wait_cta(&full[s], (kt / C::STAGES) & 1);
    const zval* Ps = reinterpret_cast<const zval*>(base + s * T::STAGE_BYTES);
    const zval* SDs = Ps + C::P_ELEMS;  // unused when C::PS == 0
    const zval* Xas = Ps + T::NP * C::P_ELEMS;
    const zval* Xbs = Xas + C::X_ELEMS;
    mb_stage_mma<C>(acc, Ps, SDs, Xas, Xbs, wm, wn, g, t);
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty[s]);
  }
  hop_epilogue_axpby<C, CM>(acc, a, i0, c0, wm, wn, g, t);
}

}  // namespace bse
