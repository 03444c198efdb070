// complex64 Chebyshev filter on the 5th-generation tensor cores (configs[4] c64 variant).
//
// FP32-accurate complex products from tcgen05.mma kind::tf32 with the 3xTF32 split
// x = hi + lo (hi = tf32(x), lo = x - hi):  a b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi.
// The operator is the same as the FP64 hop kernel (hop.cuh): with P the K-slab of [A | B],
//   U = P Xa,  L' = conj(P) Xb,  H x = [U ; -L'],
// accumulated in TMEM as [U_r | U_i] and [L'_r | L'_i] (128 lanes x 128 fp32 columns each): each
// complex product is two N = 128 UMMAs over overlapping windows of stacked X tiles
// ([-Xi | Xr | Xi] and [Xr | Xi | -Xr]), x 3 for 3xTF32.  Operands live in HBM as fp32 hi/lo
// planes in K-major layouts (P planes row-major over K, X planes = the column-major vectors) and
// are fed by 3-D TMA boxes (64-byte swizzle) whose out-of-range rows are zero-filled, so the A/B
// part and upper/lower half boundaries need no special casing.  Warp 0 = TMA producer, warp 1 =
// MMA issuer, warps 2-9 = chunked accumulation drain (round-to-nearest fp32) + epilogue:
// y+ = alpha (H y - c y) - beta y-, written back as hi/lo planes for the next step, or as raw fp32
// partials (raw mode) for the 2D grid's allreduce.  The operator may be a tile of the grid
// (output rows mo, contraction kc, the shift on a window of rows with an input offset).
// step_kernel<true> is the CTA-pair variant (cta_group::2, M = 256 over two SMs; see Geo below).
#pragma once
#include "common.cuh"
#include "tc_common.cuh"

namespace bse {
namespace c64 {

constexpr int BM = 128;               // UMMA M: output rows per CTA (per half)
constexpr int BN = 64;                // UMMA N: vector columns per CTA
constexpr int BKE = 16;               // K elements per stage (64-byte swizzle rows)
constexpr int STAGES = 2;
constexpr int CHUNK = 2;              // stages per TMEM accumulation chunk (4 UMMA K steps)
constexpr int PLANE_TILE_P = BM * BKE * 4;  // 8 KB
constexpr int PLANE_TILE_X = BN * BKE * 4;  // 4 KB
// X side per stage: for each half (a, b) and each of hi / lo a stack of three 64-row tiles,
// a: [-Xi | Xr | Xi], b: [Xr | Xi | -Xr], so that the N = 128 windows [Xr|Xi] / [-Xi|Xr] (a) and
// [Xr|Xi] / [Xi|-Xr] (b) are contiguous K-major operands
constexpr int STACK = 3 * PLANE_TILE_X;                                // 12 KB
constexpr int STAGE_BYTES = 4 * PLANE_TILE_P + 4 * STACK;              // 80 KB
constexpr int EPI_WARPS = 8;          // 2 per TMEM lane quadrant, 32 columns each
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 256;
// CTA-pair variant (cta_group::2, cluster 2 x 1 along M): the leader issues M = 256 UMMAs; each
// CTA stages its own 128 P rows and only its half of every N = 128 window, i.e. stack tiles
// [rank, rank + 1] -- 2 of the 3 -- so each SM's shared-memory operand reads per MMA drop from
// 8 KB to 6 KB (the single-CTA kernel is bound by that port).
constexpr int PAIR_STACK = 2 * PLANE_TILE_X;                           // 8 KB
constexpr int PAIR_STAGE_BYTES = 4 * PLANE_TILE_P + 4 * PAIR_STACK;    // 64 KB
constexpr int PAIR_STAGES = 3;
constexpr size_t PAIR_SMEM = 1024 + size_t(PAIR_STAGES) * PAIR_STAGE_BYTES + 256;

template <bool PAIR>
struct Geo {
  static constexpr int stages = PAIR ? PAIR_STAGES : STAGES;
  static constexpr int stage_bytes = PAIR ? PAIR_STAGE_BYTES : STAGE_BYTES;
  static constexpr int stack = PAIR ? PAIR_STACK : STACK;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// TMA into this CTA's shared memory, completing on the leader CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];\n" ::"r"(tc::smem_addr(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_addr(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc ? 1u : 0u));
}
// arrive on the barrier at this offset in both CTAs of the pair when the issued MMAs complete
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          tc::smem_addr(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// arrive on the leader CTA's copy of this barrier
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, 0;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(tc::smem_addr(bar))
      : "memory");
}

// K-major operand in the 64-byte swizzle canonical layout: rows of 64 B (16 fp32), 8-row groups
// 512 B apart; tile base 512-byte aligned.
__device__ __forceinline__ uint64_t sdesc_k_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;   // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;            // version 1
  d |= (uint64_t)4 << 61;            // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          tc::smem_addr(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

struct Maps {
  CUtensorMap p[4];  // P planes: Re hi, Re lo, Im hi, Im lo   (3-D: j, row i, part)
  CUtensorMap x[8];  // X planes of the step input: Re hi, Re lo, Im hi, Im lo, -Re hi, -Re lo, -Im hi, -Im lo
};

struct StepArgs {
  int mo, mpo;             // output rows per half, their padded half stride (multiple of 4)
  int kc, mpi;             // contraction length per part (= input rows per half), input half stride
  int k;                   // columns
  int skip_b;              // B == 0: contract over the A part only
  // planes (fp32, column-major with ld = 2 mp, lower half at row mp)
  const float* x[4];       // step input y (hi/lo, re/im; input layout) - shift operand
  const float* p[4];       // y_prev (output layout; may alias out)
  float* out[8];           // y_next (hi/lo, re/im, then the negated planes); raw: out[0] = Re, out[1] = Im
  float alpha, beta, shift;
  // the shift applies to output rows [shift_lo, shift_hi) with input row = output row + s_off
  // (a tile of the 2D grid: only the rows its input block shares with its output block)
  int shift_lo, shift_hi, s_off;
  int raw;                 // write unsplit fp32 partials (summed across the grid before the split)
};

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// hi/lo planes of (re, im) and of their negations at offset idx
__device__ __forceinline__ void store_planes(float* const (&q)[8], int64_t idx, float re, float im) {
  const float rh = tf32_hi(re), ih = tf32_hi(im), rl = re - rh, il = im - ih;
  q[0][idx] = rh;
  q[1][idx] = rl;
  q[2][idx] = ih;
  q[3][idx] = il;
  q[4][idx] = -rh;
  q[5][idx] = -rl;
  q[6][idx] = -ih;
  q[7][idx] = -il;
}

// Accumulation precision: the tensor core adds each MMA into its FP32 TMEM accumulator with
// truncation, so the error of one long accumulation grows linearly with K (measured ~2^-24 per
// add: 1.6e-4 relative at K = 8000).  The K loop is therefore cut into chunks of CHUNK stages
// accumulated in one of two TMEM buffers; the 8 epilogue warps drain each finished chunk into
// round-to-nearest FP32 register accumulators while the MMA warp fills the other buffer.
template <bool PAIR>
__global__ void __launch_bounds__(THREADS, 1) step_kernel(const __grid_constant__ Maps maps, const StepArgs a) {
  using G = Geo<PAIR>;
  constexpr int STAGES = G::stages, STAGE_BYTES = G::stage_bytes, STACK = G::stack;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base =
      smem_raw + (((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u));  // stays a shared-space pointer: LDS, not generic LD
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // column tiles fastest: a wave holds every column tile of a few row strips, so each strip of the
  // operator planes is fetched from DRAM about once (with row tiles fastest the pair variant
  // re-streamed the planes once per column tile: 262 GB per step at C3, k = 1200).
  // single CTA: grid (column tiles, row tiles); pair: grid (2 x column tiles, row-tile pairs), the
  // cluster (2, 1, 1) pairing row tiles 2y and 2y + 1 of one column tile
  const int c0 = (PAIR ? blockIdx.x / 2 : blockIdx.x) * BN;
  const int i0 = (PAIR ? 2 * blockIdx.y + (blockIdx.x & 1) : blockIdx.y) * BM;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int nk_part = (a.kc + BKE - 1) / BKE;
  const int nk = a.skip_b ? nk_part : 2 * nk_part;
  const int nchunks = (nk + CHUNK - 1) / CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], PAIR ? 2 * EPI_WARPS : EPI_WARPS);  // pair: both CTAs' drains (leader copy)
    }
    tc::fence_barrier_init();
    for (int q = 0; q < 4; ++q) {
      tc::prefetch_tmap(&maps.p[q]);
      tc::prefetch_tmap(&maps.x[q]);
    }
  }
  if (warp == 0) {  // 2 buffers x [U_r | U_i], [L'_r | L'_i] x 128 fp32 columns
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc::smem_addr(tslot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
    } else {
      tc::tmem_alloc(tslot, 512);
    }
  }
  tc::fence_before_sync();
  if constexpr (PAIR)
    cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any remote use
  else
    __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------------------------- TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const int part = kb >= nk_part;
        const int j = (kb - part * nk_part) * BKE;
        tc::mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
        if (rank == 0) tc::mbar_arrive_expect_tx(&full[s], PAIR ? 2 * STAGE_BYTES : STAGE_BYTES);
        unsigned char* st = base + s * STAGE_BYTES;
        auto load = [&](void* dst, const CUtensorMap* map, int x0, int x1, int x2) {
          if constexpr (PAIR)
            tma_load_3d_pair(dst, map, &full[s], x0, x1, x2);
          else
            tma_load_3d(dst, map, &full[s], x0, x1, x2);
        };
        for (int q = 0; q < 4; ++q) load(st + q * PLANE_TILE_P, &maps.p[q], j, i0, part);
        unsigned char* sx = st + 4 * PLANE_TILE_P;
        // Xa = half `part`, Xb = the other half (part 0: X1, X2; part 1: X2, X1)
        // plane index: re = 0 + hl, im = 2 + hl, -re = 4 + hl, -im = 6 + hl (hl: 0 hi, 1 lo)
        // a stack: [-Xi | Xr | Xi], b stack: [Xr | Xi | -Xr]; a pair CTA holds stack tiles [rank, rank + 1]
        for (int hl = 0; hl < 2; ++hl) {
          const int a_pl[3] = {6 + hl, 0 + hl, 2 + hl}, b_pl[3] = {0 + hl, 2 + hl, 4 + hl};
          unsigned char* sa = sx + hl * STACK;
          unsigned char* sb = sx + (2 + hl) * STACK;
          for (int t = 0; t < (PAIR ? 2 : 3); ++t) {
            const int tile = t + (int)rank;
            load(sa + t * PLANE_TILE_X, &maps.x[a_pl[tile]], j, part, c0);
            load(sb + t * PLANE_TILE_X, &maps.x[b_pl[tile]], j, 1 - part, c0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // -------------------------------------------------------------- MMA issuer (pair: the leader)
      constexpr uint32_t idesc = tc::idesc_tf32(PAIR ? 2 * BM : BM, 2 * BN, false, false);  // N = 128 windows
      for (int ch = 0; ch < nchunks; ++ch) {
        const int b = ch & 1;
        if (ch >= 2) tc::mbar_wait(&acc_empty[b], ((ch >> 1) - 1) & 1);
        tc::fence_after_sync();
        const uint32_t acc_u = tmem + b * 256, acc_l = acc_u + 128;  // [U_r | U_i], [L'_r | L'_i]
        const int kb_end = min(nk, (ch + 1) * CHUNK);
        for (int kb = ch * CHUNK; kb < kb_end; ++kb) {
          const int s = kb % STAGES;
          tc::mbar_wait(&full[s], (kb / STAGES) & 1);
          tc::fence_after_sync();
          const uint32_t st = tc::smem_addr(base + s * STAGE_BYTES);
          const uint32_t sx = st + 4 * PLANE_TILE_P;
#pragma unroll
          for (int kk = 0; kk < BKE / 8; ++kk) {
            const uint32_t off = kk * 32;
            const uint64_t prh = sdesc_k_sw64(st + 0 * PLANE_TILE_P + off),
                           prl = sdesc_k_sw64(st + 1 * PLANE_TILE_P + off);
            const uint64_t pih = sdesc_k_sw64(st + 2 * PLANE_TILE_P + off),
                           pil = sdesc_k_sw64(st + 3 * PLANE_TILE_P + off);
            // windows: w0 = stack rows [0, 128), w1 = rows [64, 192)
            const uint64_t a_h0 = sdesc_k_sw64(sx + 0 * STACK + off), a_h1 = sdesc_k_sw64(sx + 0 * STACK + PLANE_TILE_X + off);
            const uint64_t a_l0 = sdesc_k_sw64(sx + 1 * STACK + off), a_l1 = sdesc_k_sw64(sx + 1 * STACK + PLANE_TILE_X + off);
            const uint64_t b_h0 = sdesc_k_sw64(sx + 2 * STACK + off), b_h1 = sdesc_k_sw64(sx + 2 * STACK + PLANE_TILE_X + off);
            const uint64_t b_l0 = sdesc_k_sw64(sx + 3 * STACK + off), b_l1 = sdesc_k_sw64(sx + 3 * STACK + PLANE_TILE_X + off);
            const bool first = (kb == ch * CHUNK && kk == 0);
            // 3xTF32 real product  acc += (ph, pl) x (xh, xl)
            auto mma = [&](uint32_t acc, uint64_t pa, uint64_t xb, bool accumulate) {
              if constexpr (PAIR)
                mma_tf32_pair(acc, pa, xb, idesc, accumulate);
              else
                tc::mma_tf32(acc, pa, xb, idesc, accumulate);
            };
            auto prod = [&](uint32_t acc, uint64_t ph, uint64_t pl, uint64_t xh, uint64_t xl, bool init) {
              mma(acc, ph, xh, !init);
              mma(acc, ph, xl, true);
              mma(acc, pl, xh, true);
            };
            prod(acc_u, prh, prl, a_h1, a_l1, first);  // Pr [Xar | Xai]
            prod(acc_u, pih, pil, a_h0, a_l0, false);  // Pi [-Xai | Xar]
            prod(acc_l, prh, prl, b_h0, b_l0, first);  // Pr [Xbr | Xbi]
            prod(acc_l, pih, pil, b_h1, b_l1, false);  // Pi [Xbi | -Xbr]
          }
          if constexpr (PAIR)
            commit_pair(&empty[s]);
          else
            tc::mma_commit(&empty[s]);
        }
        if constexpr (PAIR)
          commit_pair(&acc_full[b]);
        else
          tc::mma_commit(&acc_full[b]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue warps
    const int ew = warp - 2;
    const int quad = warp & 3;          // TMEM lane quadrant this warp may access
    const int colh = ew >> 2;           // column half: 0 -> [0, 32), 1 -> [32, 64)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float acc[4][32];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[q][c] = 0.f;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int b = ch & 1;
      tc::mbar_wait(&acc_full[b], (ch >> 1) & 1);
      tc::fence_after_sync();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float v[16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tc::tmem_ld16(tmem + lane_off + b * 256 + q * 64 + colh * 32 + h * 16, v);
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[q][h * 16 + c] += v[c];
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          arrive_leader(&acc_empty[b]);
        else
          tc::mbar_arrive(&acc_empty[b]);
      }
    }
    // y+ = alpha (H y - c y) - beta y-   with  H y = [U ; -L']
    const int row = i0 + quad * 32 + lane;
    const int64_t ld = 2 * (int64_t)a.mpo, ldi = 2 * (int64_t)a.mpi;
    const bool shifted = a.shift != 0.f && row >= a.shift_lo && row < a.shift_hi;
    if (row < a.mo) {
#pragma unroll 4
      for (int c = 0; c < 32; ++c) {
        const int col = c0 + colh * 32 + c;
        if (col >= a.k) break;
        const int64_t up = (int64_t)col * ld + row, lo = up + a.mpo;
        float hur = acc[0][c], hui = acc[1][c], hlr = -acc[2][c], hli = -acc[3][c];
        if (shifted) {
          const int64_t xu = (int64_t)col * ldi + row + a.s_off, xl = xu + a.mpi;
          hur -= a.shift * (a.x[0][xu] + a.x[1][xu]);
          hui -= a.shift * (a.x[2][xu] + a.x[3][xu]);
          hlr -= a.shift * (a.x[0][xl] + a.x[1][xl]);
          hli -= a.shift * (a.x[2][xl] + a.x[3][xl]);
        }
        float yur = a.alpha * hur, yui = a.alpha * hui, ylr = a.alpha * hlr, yli = a.alpha * hli;
        if (a.beta != 0.f) {
          yur -= a.beta * (a.p[0][up] + a.p[1][up]);
          yui -= a.beta * (a.p[2][up] + a.p[3][up]);
          ylr -= a.beta * (a.p[0][lo] + a.p[1][lo]);
          yli -= a.beta * (a.p[2][lo] + a.p[3][lo]);
        }
        if (a.raw) {
          a.out[0][up] = yur;
          a.out[1][up] = yui;
          a.out[0][lo] = ylr;
          a.out[1][lo] = yli;
        } else {
          store_planes(a.out, up, yur, yui);
          store_planes(a.out, lo, ylr, yli);
        }
      }
    }
  }
  tc::fence_before_sync();
  if constexpr (PAIR) {
    cluster_sync();  // the leader's MMAs wrote this CTA's TMEM, the peer's arrivals hit the leader
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  } else {
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- layout conversions
// P planes of an operator tile with output rows i < mo and contraction index j < kc per part:
// plane[q][i * (2 mp) + part * mp + j] = hi/lo of Re/Im P[i, part, j], mp = pad4(kc).  The rows are
// read as columns of the *transposed* blocks src_a / src_b (column-major, leading dim lds, column i
// = entries j): P_A[i, j] = conj(src_a[j, i]) (A^H block), P_B[i, j] = src_b[j, i] (B^T block).
// One GPU: src = [A | B] itself (A hermitian, B symmetric); 2D grid: the fwd tile's planes come
// from the trn tile's columns and vice versa.  Coalesced reads and writes.
__global__ void p_planes_kernel(const zval* __restrict__ src_a, const zval* __restrict__ src_b, int64_t lds, int mo,
                                int kc, int mp, float* __restrict__ pl0, float* __restrict__ pl1,
                                float* __restrict__ pl2, float* __restrict__ pl3) {
  const int64_t total = (int64_t)mo * 2 * mp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / (2 * mp);
    const int J = int(idx % (2 * mp));
    const int part = J >= mp, j = J - part * mp;
    float re = 0.f, im = 0.f;
    if (j < kc) {
      const zval v = (part ? src_b : src_a)[i * lds + j];  // column i of the transposed block, entry j
      re = (float)v.re;
      im = part ? (float)v.im : -(float)v.im;
    }
    const float rh = tf32_hi(re), ih = tf32_hi(im);
    pl0[idx] = rh;
    pl1[idx] = re - rh;
    pl2[idx] = ih;
    pl3[idx] = im - ih;
  }
}

struct Planes8 {
  float* p[8];
};

// c128 vectors (n x k, ldv) -> hi/lo planes (ld = 2 mp, lower half at mp; pad rows zero)
__global__ void to_planes_kernel(const zval* __restrict__ v, int64_t ldv, int m, int mp, int k, Planes8 q) {
  const int64_t ld = 2 * (int64_t)mp, total = ld * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = idx / ld;
    const int r = int(idx % ld);
    const int half = r >= mp, rr = r - half * mp;
    float re = 0.f, im = 0.f;
    if (rr < m) {
      const zval z = v[col * ldv + half * m + rr];
      re = (float)z.re;
      im = (float)z.im;
    }
    store_planes(q.p, idx, re, im);
  }
}

// raw fp32 (re, im) partial sums (ld = 2 mp) -> the 8 hi/lo planes of the next step's input
__global__ void split_planes_kernel(const float* __restrict__ re, const float* __restrict__ im, int m, int mp, int k,
                                    Planes8 q) {
  const int64_t ld = 2 * (int64_t)mp, total = ld * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = int(idx % ld);
    const int rr = r >= mp ? r - mp : r;
    store_planes(q.p, idx, rr < m ? re[idx] : 0.f, rr < m ? im[idx] : 0.f);
  }
}

__global__ void from_planes_kernel(const float* __restrict__ q0, const float* __restrict__ q1,
                                   const float* __restrict__ q2, const float* __restrict__ q3, int m, int mp, int k,
                                   zval* __restrict__ v, int64_t ldv) {
  const int64_t n = 2 * (int64_t)m, total = n * k, ld = 2 * (int64_t)mp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = idx / n;
    const int r = int(idx % n);
    const int half = r >= m, rr = r - half * m;
    const int64_t s = col * ld + half * mp + rr;
    v[col * ldv + r] = zval{(double)q0[s] + (double)q1[s], (double)q2[s] + (double)q3[s]};
  }
}

}  // namespace c64
}  // namespace bse
