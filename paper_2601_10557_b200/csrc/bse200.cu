// bse200: C ABI of the B200-native pseudo-hermitian ChASE hot path.
// See include/bse200.h for the contract and DESIGN.md for the data layout.
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <ctime>
#include <mutex>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/bse200.h"
#include "aux.cuh"
#include "c64.cuh"
#include "hop.cuh"
#include "hop_mb.cuh"
#include "hop_rs.cuh"
#include "zgemm.cuh"

using bse::zval;

// ----------------------------------------------------------------------------
// context, errors, workspace
// ----------------------------------------------------------------------------
struct bse_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cusolverDnParams_t params = nullptr;
  std::string err;
  int64_t launches = 0;
  void* ws = nullptr;  // general device scratch
  // real-split planes registered for the RR products of one operator (bse_set_rs_planes)
  const void* rs_ab = nullptr;
  const double* rs_g = nullptr;
  int64_t rs_ldg = 0, rs_m = 0;
  // optional capture of the RR's k x k reduced problem (bse_set_rr_capture): [W | L | M | G] + d
  zval* rr_capture = nullptr;
  size_t ws_bytes = 0;
  void* hws = nullptr;  // host scratch (cuSOLVER 64-bit API)
  size_t hws_bytes = 0;
  double* pinned = nullptr;  // pinned host staging (small results)
  size_t pinned_count = 0;
  int filter_cm = 4;  // complex multiplication of the Chebyshev products: 4 (4M) or 3 (3M / Gauss)
  void* sws = nullptr;  // persistent cuSOLVER device workspace (grows, never shrinks)
  size_t sws_bytes = 0;
  unsigned ham_flags = 0;  // BSE_HAM_B_ZERO: operator calls skip the B half of the contraction
  int rs_group_rows = 8;  // real-split CTA raster (hop_rs.cuh): BSE200_RS_GROUP_ROWS, 0 = columns fastest
  int rs_ksplit = 0;      // real-split split-K: BSE200_RS_KSPLIT (0 = planned per product, rs_plan)
  int push_n = 0;         // fused group reduction: push targets of the next real-split products
  zval* push_base[4] = {nullptr, nullptr, nullptr, nullptr};
  void* gv = nullptr;  // split-K GEMV partials
  size_t gv_bytes = 0;
  // second stream + cuSOLVER handle: the RR pencil's eigenvalues of M run beside chol(W) -> eigh(G)
  cudaStream_t aux = nullptr;
  cusolverDnHandle_t aux_solver = nullptr;
  cusolverDnParams_t aux_params = nullptr;
  void* aux_dws = nullptr;
  size_t aux_dws_bytes = 0;
  void* aux_hws = nullptr;
  size_t aux_hws_bytes = 0;
  double* aux_pinned = nullptr;
  size_t aux_pinned_count = 0;
  cudaEvent_t aux_ev[2] = {nullptr, nullptr};
};

namespace {

struct BseError : std::runtime_error {
  int code;
  BseError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(x)                                                                                    \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess)                                                                            \
      throw BseError(BSE_ECUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " at " #x);     \
  } while (0)
#define BLAS_OK(x)                                                                                    \
  do {                                                                                                \
    cublasStatus_t s_ = (x);                                                                          \
    if (s_ != CUBLAS_STATUS_SUCCESS) throw BseError(BSE_ECUDA, "cuBLAS status " + std::to_string(s_) + " at " #x); \
  } while (0)
#define SOLVER_OK(x)                                                                                  \
  do {                                                                                                \
    cusolverStatus_t s_ = (x);                                                                        \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                \
      throw BseError(BSE_ECUDA, "cuSOLVER status " + std::to_string(s_) + " at " #x);                 \
  } while (0)

// cudaFuncSetAttribute applies per device (context): remember the (kernel, device) pairs already
// raised, under a lock, so a second GPU driven from the same process gets its own call.
void ensure_smem(bse_ctx* ctx, const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, ctx->device})) return;
  CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({fn, ctx->device});
}

void check_launch(bse_ctx* ctx) {
  ctx->launches++;
  CUDA_OK(cudaGetLastError());
}

template <class F>
int guarded(bse_ctx* ctx, F&& f) {
  if (!ctx) return BSE_EVALIDATION;
  try {
    CUDA_OK(cudaSetDevice(ctx->device));
    f();
    ctx->err.clear();
    return BSE_OK;
  } catch (const BseError& e) {
    ctx->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return BSE_ECUDA;
  }
}

// Bump allocator over the context workspace.  ensure() must be called with the
// call's total need before any carve (it may reallocate, which synchronises).
struct Scratch {
  bse_ctx* ctx;
  size_t off = 0;
  explicit Scratch(bse_ctx* c, size_t total) : ctx(c) {
    total += 4096;
    if (ctx->ws_bytes < total) {
      if (ctx->ws) {
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        CUDA_OK(cudaFree(ctx->ws));
      }
      const size_t want = std::max(total, ctx->ws_bytes * 3 / 2);
      ctx->ws = nullptr;
      ctx->ws_bytes = 0;
      CUDA_OK(cudaMalloc(&ctx->ws, want));
      ctx->ws_bytes = want;
    }
  }
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(static_cast<char*>(ctx->ws) + off);
    off += count * sizeof(T);
    if (off > ctx->ws_bytes) throw BseError(BSE_ECUDA, "internal: workspace overrun");
    return p;
  }
};

inline size_t al(size_t bytes) { return (bytes + 255) & ~size_t(255); }

// Opt-in step timer (BSE200_TIMING=1): synchronises the stream at each mark and prints the wall
// time of every step of an entry point to stderr.  Off by default (no syncs added).
struct StepTimer {
  bse_ctx* ctx;
  const char* name;
  bool on;
  double t0, tl;
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
  }
  StepTimer(bse_ctx* c, const char* n) : ctx(c), name(n) {
    const char* e = getenv("BSE200_TIMING");
    on = e && e[0] == '1';
    if (on) {
      cudaStreamSynchronize(ctx->stream);
      t0 = tl = now();
    }
  }
  void mark(const char* step, int64_t k = -1) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const double t = now();
    fprintf(stderr, "[bse200 %s k=%lld] %-22s %8.2f ms\n", name, (long long)k, step, 1e3 * (t - tl));
    tl = t;
  }
};

double* pinned(bse_ctx* ctx, size_t count) {
  if (ctx->pinned_count < count) {
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    CUDA_OK(cudaMallocHost(&ctx->pinned, count * sizeof(double)));
    ctx->pinned_count = count;
  }
  return ctx->pinned;
}

// Persistent device workspace for cuSOLVER: allocated once per size high-water mark, so the
// k x k factorisations never touch an allocator inside the iteration (stream-ordered
// cudaMallocAsync/cudaFreeAsync pairs caused 0.2-1.7 s host stalls at C3, profiles/r01/).
void* solver_ws(bse_ctx* ctx, size_t bytes) {
  bytes = std::max<size_t>(bytes, 256);
  if (ctx->sws_bytes < bytes) {
    const size_t want = std::max(bytes, ctx->sws_bytes * 3 / 2);
    if (ctx->sws) {
      CUDA_OK(cudaStreamSynchronize(ctx->stream));
      CUDA_OK(cudaFree(ctx->sws));
    }
    ctx->sws = nullptr;
    ctx->sws_bytes = 0;
    CUDA_OK(cudaMalloc(&ctx->sws, want));
    ctx->sws_bytes = want;
  }
  return ctx->sws;
}

void* host_ws(bse_ctx* ctx, size_t bytes) {
  if (ctx->hws_bytes < bytes) {
    free(ctx->hws);
    ctx->hws = malloc(bytes);
    ctx->hws_bytes = bytes;
  }
  return ctx->hws;
}

inline int grid1d(int64_t n, int threads = 256, int cap = 148 * 16) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

// ----------------------------------------------------------------------------
// H operator launches
// ----------------------------------------------------------------------------
// Tile configuration of the fused H-operator GEMM:
// CTA 64 x 32 complex (up and low halves), 8 warps of 16 x 16, BK = 8, 4 stages.
using HopMain = bse::HopCfg<64, 32, 8, 2, 2, 4, 2>;
// 3M (Gauss) variant: 6 accumulators per block pair -> one 8-warp CTA per SM, deeper K stages
using Hop3M = bse::HopCfg<64, 32, 16, 2, 2, 4, 1>;

template <class C, int EPI, int CM = 4>
void launch_hop(bse_ctx* ctx, const bse::HopArgs& a_in) {
  bse::HopArgs a = a_in;
  a.skip_b = (ctx->ham_flags & BSE_HAM_B_ZERO) ? 1 : 0;
  ensure_smem(ctx, (const void*)bse::hop_kernel<C, EPI, CM>, (int)C::SMEM);
  dim3 grid((a.k + C::BN - 1) / C::BN, (a.mr + C::BM - 1) / C::BM);
  bse::hop_kernel<C, EPI, CM><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(a);
  check_launch(ctx);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw BseError(BSE_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D FP64 tensor map, no swizzle (the box rows carry their own padding, hop_mb.cuh)
CUtensorMap map2d_f64(const void* base, uint64_t d0, uint64_t d1, uint64_t stride1_bytes, uint32_t b0, uint32_t b1) {
  CUtensorMap map;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {stride1_bytes};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw BseError(BSE_ECUDA, "cuTensorMapEncodeTiled (f64) failed (" + std::to_string((int)r) + ")");
  return map;
}

template <class C>
void launch_hop_tma(bse_ctx* ctx, const bse::HopArgs& a_in) {
  bse::HopArgs a = a_in;
  a.skip_b = (ctx->ham_flags & BSE_HAM_B_ZERO) ? 1 : 0;
  constexpr size_t smem = bse::TmaLayout<C>::SMEM;
  ensure_smem(ctx, (const void*)bse::hop3m_tma_kernel<C>, (int)smem);
  bse::HopMaps mp;
  const uint64_t pr = 2 * (uint64_t)a.mr, xr = 2 * (uint64_t)a.kc;
  const zval* pp[2] = {a.pa, a.pb};
  const zval* ss[2] = {a.sa, a.sb};
  const zval* xx[2] = {a.x1, a.x2};
  for (int q = 0; q < 2; ++q) {
    mp.p[q] = map2d_f64(pp[q], pr, a.kc, a.lda * 16, 2 * (C::BM + 2), C::BK);
    mp.sd[q] = C::PS ? map2d_f64(ss[q], pr, a.kc, a.lda * 16, 2 * (C::BM + 2), C::BK) : mp.p[q];
    mp.x[q] = map2d_f64(xx[q], xr, a.k, a.ldx * 16, 2 * (C::BK + 4), C::BN);
  }
  dim3 grid((a.k + C::BN - 1) / C::BN, (a.mr + C::BM - 1) / C::BM);
  bse::hop3m_tma_kernel<C><<<grid, C::THREADS + 32, smem, ctx->stream>>>(a, mp);
  check_launch(ctx);
}


// Filter-product variants (bse_set_filter_algorithm codes; the sweeps that chose them are in
// profiles/r01/tune_*.txt):
//   88  default 3M: TMA-fed, producer warp, mbarrier rings (hop_mb.cuh); tile by block width
//   82 / 86  its two tiles alone (64 x 16, 4 consumer warps, 2 CTAs/SM / 64 x 32, 8 warps, 6 stages)
//    4  4M (HopMain)
// (round 1's dominated 3M feeds -- cp.async + mbarrier, cp.async + __syncthreads, sums in
// registers through hop_kernel -- are retired; profiles/r01/tune_3m_*.txt keeps their numbers)
using Hop3MNarrow = bse::HopCfg<64, 16, 8, 4, 1, 4, 2, 1>;
using Hop3MWide = bse::HopCfg<64, 32, 8, 4, 1, 6, 1, 1>;
// the default's tiles without sum planes (HBM too short for them): operand sums formed in registers
using Hop3MNarrowNP = bse::HopCfg<64, 16, 8, 4, 1, 4, 2, 0>;
using Hop3MWideNP = bse::HopCfg<64, 32, 8, 4, 1, 6, 1, 0>;

// 90 (92 / 94 / 96 / 97 / 98): the real-split kernel (hop_rs.cuh) -- bse_chebyshev_filter_rs, the RR's S H Q
// on registered planes, the grid's tile products (bse_hop_tile_rs / _rs_t); the complex-operand
// products that remain (B = 0, no planes) run code 88 under it
bool filter_code_needs_planes(int code) {
  return code == 82 || code == 86 || code == 88 || code == 90 || code == 92 || code == 94 || code == 96 || code == 97 ||
         code == 98;
}
bool filter_code_valid(int code) { return code == 4 || filter_code_needs_planes(code); }

// Chebyshev-step products, as selected by bse_set_filter_algorithm
void launch_filter_hop(bse_ctx* ctx, const bse::HopArgs& a) {
  int code = ctx->filter_cm >= 90 ? 88 : ctx->filter_cm;
  if (filter_code_needs_planes(code) && (!a.sa || !a.sb))  // no P sum planes: sums in registers
    code = -88;  // internal only (not a bse_set_filter_algorithm code)
  switch (code) {
    case -88:  // the default's TMA kernel forming the operand sums in registers (same bits)
      if (a.k >= 512)
        launch_hop_tma<Hop3MWideNP>(ctx, a);
      else
        launch_hop_tma<Hop3MNarrowNP>(ctx, a);
      break;
    // default 3M: 64 x 32 CTA (8 consumer warps, 6 stages) for wide blocks, 64 x 16 (4 warps,
    // 2 CTAs/SM) below 512 columns where the wider tile underfills the GPU.  Every variant
    // accumulates each output in the same K order: the choice never changes a bit.
    case 88:
      if (a.k >= 512)
        launch_hop_tma<Hop3MWide>(ctx, a);
      else
        launch_hop_tma<Hop3MNarrow>(ctx, a);
      break;
    case 82: launch_hop_tma<Hop3MNarrow>(ctx, a); break;
    case 86: launch_hop_tma<Hop3MWide>(ctx, a); break;
    default: launch_hop<HopMain, bse::HOP_AXPBY, 4>(ctx, a); break;
  }
}

// ---- real-split filter (hop_rs.cuh) ----
// tiles (codes for bse_set_filter_algorithm; 90 picks 97 or 94, and a split-K factor, by rs_plan below):
//   97  128 x 32, 4 consumer warps of 32 x 32, BK = 32 double buffered, 2 CTAs / SM -- 96.8% of the
//       DMMA peak at m = 20k, k = 1200 in both directions (profiles/r02/rs_tall4_bk32.txt)
//   96  the same with BK = 16, 3 stages (95.3%)
//   92  128 x 32, 8 consumer warps of 32 x 16, 6 stages, 1 CTA / SM (round-1 default: 92.6%)
//   94  64 x 32, 8 consumer warps of 16 x 16, 5 stages, 2 CTAs / SM: twice the CTAs, so the better
//       one when the 128-row tile leaves a short last wave (small k or small tiles of the 2D grid)
using RsTall = bse::RsCfg<128, 32, 16, 4, 2, 6, 1>;
using RsNarrow = bse::RsCfg<64, 32, 16, 2, 2, 5, 2>;
using RsTall4 = bse::RsCfg<128, 32, 16, 4, 4, 3, 2>;
using RsTall4K32 = bse::RsCfg<128, 32, 32, 4, 4, 2, 2>;

// Default plan: the 128-row 4-warp tile runs at ~96.8% of the DMMA peak in full waves, the 64-row
// tile at ~93.5%; each is discounted by the fill of its last wave (2 resident CTAs per SM).  A short
// last wave (the 10k-row tiles of a 2 x 2 grid, small k late in the solve) can instead be filled by
// splitting each tile's K range over ksplit CTAs: the partial sums cost 2 ksplit k rows 16 B of HBM
// traffic (written once, read once by rs_splitk_epilogue_kernel) plus one extra launch.
struct RsPlan {
  bool wide;
  int ksplit;
};
constexpr size_t RS_SPLIT_WS_MAX = size_t(2) << 30;  // cap on the split-K partials (ctx->gv)

RsPlan rs_plan(int64_t rows, int64_t kc, int64_t k, int force_split = 0) {
  const double slots = 148.0 * 2;
  const double col = double((k + 31) / 32);
  const double flop_s = 16.0 * double(rows) * double(kc) * double(k) / 37.1e12;  // at the DMMA peak
  RsPlan best{true, 1};
  double best_t = 1e300;
  for (int wide = 1; wide >= 0; --wide) {
    const int64_t bm = wide ? 128 : 64;
    const double eff = wide ? 0.968 : 0.935;
    const int64_t nkt = 2 * ((kc + 31) / 32);  // K stages of a tile (BK 32; the 64-row tile's BK 16 doubles it)
    const double waves1 = col * 2.0 * double((rows + bm - 1) / bm) / slots;
    const bool can_split = nkt / 2 >= 16 && (size_t)2 * 2 * k * rows * 16 <= RS_SPLIT_WS_MAX;
    for (int sp = 1; sp <= 4; ++sp) {
      if (force_split > 0 && sp != force_split) continue;
      if (sp > 1 && (nkt / sp < 16 || (size_t)sp * 2 * k * rows * 16 > RS_SPLIT_WS_MAX)) continue;
      // under ~20 waves the unsplit grid loses more to the uneven finish of its long CTAs than
      // the fill estimate shows (m = 10k: k = 810 93.9% unsplit vs 95.1% split 4, k = 266
      // 86.3% vs 90.7%; profiles/r02/rs_plan_m10k.txt)
      if (sp == 1 && force_split == 0 && waves1 < 20.0 && can_split) continue;
      const double waves = waves1 * sp;
      double t = flop_s / eff * std::ceil(waves) / waves;
      if (sp > 1) t += (2.0 * sp * 2.0 * double(k) * double(rows) * 16.0) / 6.0e12 + 4e-6;
      if (t < best_t * 0.995) {  // prefer the earlier (wider, unsplit) plan on near ties
        best_t = t;
        best = RsPlan{wide == 1, sp};
      }
    }
  }
  return best;
}

// the split-K partial buffer (shared with launch_gemv: never live at the same time)
void* ensure_gv(bse_ctx* ctx, size_t need) {
  if (ctx->gv_bytes < need) {
    if (ctx->gv) {
      CUDA_OK(cudaStreamSynchronize(ctx->stream));
      CUDA_OK(cudaFree(ctx->gv));
    }
    ctx->gv = nullptr;
    ctx->gv_bytes = 0;
    CUDA_OK(cudaMalloc(&ctx->gv, need));
    ctx->gv_bytes = need;
  }
  return ctx->gv;
}

// TRANS: the transposed-tile product on the same planes (hop_rs.cuh header): a.mr output rows
// = plane columns, a.kc contraction = plane rows; the planes are read through K-major boxes.
template <class C, bool TRANS = false, bool GENERIC = false>
void launch_rs(bse_ctx* ctx, const bse::HopArgs& a, const double* g, int64_t ldg, int ksplit = 1) {
  constexpr size_t smem = C::template smem<TRANS>();
  // fused group reduction: the PUSH instantiation stores the output tiles to the push targets;
  // split-K products push from rs_splitk_epilogue_kernel instead
  const bool push = ctx->push_n > 0 && ksplit == 1;
  if (push)
    ensure_smem(ctx, (const void*)bse::hop_rs_tma_kernel<C, TRANS, GENERIC, true>, (int)smem);
  else
    ensure_smem(ctx, (const void*)bse::hop_rs_tma_kernel<C, TRANS, GENERIC>, (int)smem);
  bse::RsMaps mp;
  for (int q = 0; q < 4; ++q) {
    if (TRANS)
      mp.g[q] = map2d_f64(g + (int64_t)q * a.mr * ldg, a.kc, a.mr, ldg * 8, C::LDK, C::BM);
    else
      mp.g[q] = map2d_f64(g + (int64_t)q * a.kc * ldg, a.mr, a.kc, ldg * 8, C::LDP, C::BK);
  }
  mp.x[0] = map2d_f64(a.x1, 2 * (uint64_t)a.kc, a.k, a.ldx * 16, 2 * C::LDX, C::BN);
  mp.x[1] = map2d_f64(a.x2, 2 * (uint64_t)a.kc, a.k, a.ldx * 16, 2 * C::LDX, C::BN);
  const int nbm = (a.mr + C::BM - 1) / C::BM;
  dim3 grid((a.k + C::BN - 1) / C::BN, 2 * nbm, ksplit);
  bse::HopArgs ar = a;
  ar.group_rows = ctx->rs_group_rows;
  ar.ksplit = ksplit;
  ar.part_ws = nullptr;
  ar.npush = ctx->push_n;
  for (int r = 0; r < 4; ++r) ar.push[r] = ctx->push_base[r];
  if (ksplit > 1)
    ar.part_ws = static_cast<zval*>(ensure_gv(ctx, (size_t)ksplit * 2 * a.k * a.mr * sizeof(zval)));
  if (push)
    bse::hop_rs_tma_kernel<C, TRANS, GENERIC, true><<<grid, C::THREADS + 32, smem, ctx->stream>>>(ar, mp);
  else
    bse::hop_rs_tma_kernel<C, TRANS, GENERIC><<<grid, C::THREADS + 32, smem, ctx->stream>>>(ar, mp);
  check_launch(ctx);
  if (ksplit > 1) {
    const int64_t total = 2 * (int64_t)a.k * a.mr;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    bse::rs_splitk_epilogue_kernel<<<blocks, 256, 0, ctx->stream>>>(ar);
    check_launch(ctx);
  }
}

// one real-split product (folded input x1 / x2, output halves y1 / y2) on the tile's planes g
// the 8-warp 128 x 32 tile reads its fragments through generic loads, the others through LDS (the
// faster of each, profiles/r02/rs_consumer_variants_*.txt, rs_tall4_*.txt); all bitwise identical
template <bool TRANS = false>
void rs_product(bse_ctx* ctx, const bse::HopArgs& a, const double* g, int64_t ldg) {
  switch (ctx->filter_cm) {
    case 92: launch_rs<RsTall, TRANS, true>(ctx, a, g, ldg); break;
    case 94: launch_rs<RsNarrow, TRANS, false>(ctx, a, g, ldg); break;
    case 96: launch_rs<RsTall4, TRANS, false>(ctx, a, g, ldg); break;
    case 97: launch_rs<RsTall4K32, TRANS, false>(ctx, a, g, ldg); break;
    case 98: launch_rs<RsTall4K32, TRANS, false>(ctx, a, g, ldg, ctx->rs_ksplit > 1 ? ctx->rs_ksplit : 2); break;
    default: {
      const RsPlan p = rs_plan(a.mr, a.kc, a.k, ctx->rs_ksplit);
      if (p.wide)
        launch_rs<RsTall4K32, TRANS, false>(ctx, a, g, ldg, p.ksplit);
      else
        launch_rs<RsNarrow, TRANS, false>(ctx, a, g, ldg, p.ksplit);
    }
  }
}

bse::HopArgs hop_args_single(const void* d_ab, int64_t lda, int64_t m, const zval* x, int64_t ldx, int64_t k);

void rs_step(bse_ctx* ctx, const double* g, int64_t ldg, int64_t m, const zval* cur, const zval* prev, zval* next,
             int64_t ld, int64_t k, double c, double alpha, double beta) {
  bse::HopArgs a = hop_args_single(nullptr, m, m, cur, ld, k);
  a.y1 = next;
  a.y2 = next + m;
  a.ldy = ld;
  a.s1 = cur;
  a.s2 = cur + m;
  a.lds = ld;
  a.shift = c;
  a.alpha = alpha;
  a.beta = beta;
  if (beta != 0.0) {
    a.p1 = prev;
    a.p2 = prev + m;
    a.ldp = ld;
  }
  rs_product(ctx, a, g, ldg);
}

// k == 1 products (Lanczos): split-K GEMV, partials in the context workspace tail
void launch_gemv(bse_ctx* ctx, const bse::HopArgs& a) {
  const int rb = (a.mr + bse::GV_THREADS - 1) / bse::GV_THREADS;
  int nsplit = std::max(1, std::min(64, (148 * 8 + rb - 1) / rb));
  nsplit = std::min(nsplit, std::max(1, a.kc / 64));
  const int kchunk = (a.kc + nsplit - 1) / nsplit;
  zval* part = static_cast<zval*>(ensure_gv(ctx, (size_t)nsplit * 2 * a.mr * sizeof(zval)));
  bse::gemv_partial_kernel<<<dim3(rb, nsplit), bse::GV_THREADS, 0, ctx->stream>>>(
      a.pa, a.pb, a.lda, a.mr, a.kc, a.x1, a.x2, kchunk, part, (ctx->ham_flags & BSE_HAM_B_ZERO) ? 1 : 0);
  check_launch(ctx);
  bse::gemv_reduce_kernel<<<(2 * a.mr + 255) / 256, 256, 0, ctx->stream>>>(part, nsplit, a.mr, a.y1, a.y2, a.alpha,
                                                                           a.low_sign);
  check_launch(ctx);
}

bse::HopArgs hop_args_single(const void* d_ab, int64_t lda, int64_t m, const zval* x, int64_t ldx, int64_t k) {
  bse::HopArgs a{};
  const zval* ab = static_cast<const zval*>(d_ab);
  a.pa = ab;
  a.pb = ab ? ab + m * lda : nullptr;  // null for the real-split products (planes passed separately)
  a.lda = lda;
  a.mr = (int)m;
  a.kc = (int)m;
  a.x1 = x;
  a.x2 = x + m;
  a.ldx = ldx;
  a.k = (int)k;
  a.alpha = 1.0;
  a.beta = 0.0;
  a.shift = 0.0;
  a.low_sign = 1.0;
  a.shift_lo = 0;
  a.shift_hi = (int)m;
  a.shift_col = nullptr;
  return a;
}

void launch_filter_hop(bse_ctx* ctx, const bse::HopArgs& a);

bool rs_active(const bse_ctx* ctx, const void* d_ab, int64_t m) {
  return ctx->rs_g && ctx->rs_ab == d_ab && ctx->rs_m == m && !(ctx->ham_flags & BSE_HAM_B_ZERO);
}

// y = H x / S H x; with the sum planes d_sd the product takes the filter kernel (3M), else 4M;
// with real-split planes registered for d_ab and a fold buffer (n x k, ld n) the real-split kernel
void apply_h(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, const zval* x, int64_t ldx, zval* y, int64_t ldy,
             int64_t k, double low_sign, const void* d_sd = nullptr, zval* fold = nullptr) {
  if (k == 0 || m == 0) return;
  // k == 1 takes the GEMV on [A|B] unless the operator is held as planes only (d_ab == NULL)
  if ((k > 1 || !d_ab) && fold && rs_active(ctx, d_ab, m)) {
    const int fb = grid1d(m * k, 256, 148 * 16);
    // fold x into the buffer, the product into y's halves, then unfold y in place (with the S-flip)
    bse::rs_fold_kernel<<<fb, 256, 0, ctx->stream>>>(x, fold, ldx, 2 * m, m, k, 1.0, 1.0);
    check_launch(ctx);
    bse::HopArgs a = hop_args_single(d_ab, lda, m, fold, 2 * m, k);
    a.y1 = y;
    a.y2 = y + m;
    a.ldy = ldy;
    rs_product(ctx, a, ctx->rs_g, ctx->rs_ldg);
    bse::rs_fold_kernel<<<fb, 256, 0, ctx->stream>>>(y, y, ldy, ldy, m, k, 0.5, 0.5 * low_sign);
    check_launch(ctx);
    return;
  }
  bse::HopArgs a = hop_args_single(d_ab, lda, m, x, ldx, k);
  a.y1 = y;
  a.y2 = y + m;
  a.ldy = ldy;
  a.low_sign = low_sign;
  if (k == 1) {
    launch_gemv(ctx, a);
  } else if (d_sd) {
    a.sa = static_cast<const zval*>(d_sd);
    a.sb = a.sa + m * lda;
    launch_filter_hop(ctx, a);
  } else {
    launch_hop<HopMain, bse::HOP_AXPBY>(ctx, a);
  }
}

void filter_step(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const zval* y,
                 const zval* yprev, zval* ynext, int64_t ld, int64_t k, double c, double alpha, double beta) {
  bse::HopArgs a = hop_args_single(d_ab, lda, m, y, ld, k);
  if (d_sd) {
    a.sa = static_cast<const zval*>(d_sd);
    a.sb = a.sa + m * lda;
  }
  a.y1 = ynext;
  a.y2 = ynext + m;
  a.ldy = ld;
  a.s1 = y;
  a.s2 = y + m;
  a.lds = ld;
  a.shift = c;
  a.alpha = alpha;
  a.beta = beta;
  if (beta != 0.0) {
    a.p1 = yprev;
    a.p2 = yprev + m;
    a.ldp = ld;
  }
  launch_filter_hop(ctx, a);
}

// residual norms into d_out (k doubles, device)
void residual_norms(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, const zval* v, int64_t ldv, int64_t k,
                    const double* d_lam, double* d_part, double* d_out) {
  bse::HopArgs a = hop_args_single(d_ab, lda, m, v, ldv, k);
  a.s1 = v;
  a.s2 = v + m;
  a.lds = ldv;
  a.lam = d_lam;
  a.partial = d_part;
  launch_hop<HopMain, bse::HOP_RESID>(ctx, a);
  const int nb = (int)((m + HopMain::BM - 1) / HopMain::BM);
  bse::resid_finalize_kernel<<<(int)((k + 127) / 128), 128, 0, ctx->stream>>>(d_part, nb, (int)k, d_out);
  check_launch(ctx);
}

size_t resid_part_count(int64_t m, int64_t k) { return (size_t)((m + HopMain::BM - 1) / HopMain::BM) * k; }

// ----------------------------------------------------------------------------
// GEMMs
// ----------------------------------------------------------------------------
using GemmMain = bse::GemmCfg<64, 64, 8, 4, 2, 4>;

// Split-K factor: enough CTAs to fill the GPU and little wave quantisation (the last wave of a
// 361-tile Gram at k = 1200 ran 78% idle without a split), keeping >= 16 k-tiles per split.
int splitk_for(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + GemmMain::BM - 1) / GemmMain::BM) * ((N + GemmMain::BN - 1) / GemmMain::BN);
  const int64_t slots = 148 * 2;  // resident CTAs (2 per SM)
  const int64_t kt = (K + GemmMain::BK - 1) / GemmMain::BK;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, kt / 16));
  auto fill = [&](int64_t s) {  // fraction of the launched waves' CTA slots that do work
    const int64_t ctas = tiles * s;
    return (double)ctas / (double)(((ctas + slots - 1) / slots) * slots);
  };
  if (tiles >= 8 * slots || fill(1) >= 0.9) return 1;  // many waves: quantisation is negligible
  int64_t best = 1;
  for (int64_t s = 1; s <= smax; ++s) {
    if (tiles * s >= slots && fill(s) >= 0.9) return (int)s;
    if (fill(s) > fill(best) + 1e-9) best = s;
  }
  return (int)best;
}

size_t gemm_ws_bytes(int64_t M, int64_t N, int64_t K) {
  const int s = splitk_for(M, N, K);
  return s > 1 ? al((size_t)s * M * N * sizeof(zval)) : 0;
}

template <int OPA>
void zgemm(bse_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const zval* a, int64_t lda, const zval* b,
           int64_t ldb, double beta, zval* c, int64_t ldc, zval* ws, int tri = 0) {
  if (M == 0 || N == 0) return;
  using C = GemmMain;
  ensure_smem(ctx, (const void*)bse::zgemm_kernel<C, OPA>, (int)C::SMEM);
  bse::GemmArgs g{};
  g.a = a;
  g.lda = lda;
  g.b = b;
  g.ldb = ldb;
  g.c = c;
  g.ldc = ldc;
  g.M = (int)M;
  g.N = (int)N;
  g.K = (int)K;
  g.alpha = alpha;
  g.beta = beta;
  g.tri = tri;
  const int splits = (K == 0) ? 1 : splitk_for(M, N, K);
  g.ws = ws;
  if (splits > 1 && !ws) throw BseError(BSE_ECUDA, "internal: split-K workspace missing");
  dim3 grid((unsigned)((M + C::BM - 1) / C::BM), (unsigned)((N + C::BN - 1) / C::BN), (unsigned)splits);
  bse::zgemm_kernel<C, OPA><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(g);
  check_launch(ctx);
  if (splits > 1) {
    bse::zgemm_splitk_reduce<<<grid1d(M * N), 256, 0, ctx->stream>>>(ws, splits, c, ldc, (int)M, (int)N, alpha, beta,
                                                                     tri);
    check_launch(ctx);
  }
}

// ----------------------------------------------------------------------------
// small dense pieces (k x k) on device: cuSOLVER / cuBLAS
// ----------------------------------------------------------------------------
const cuDoubleComplex* cz(const zval* p) { return reinterpret_cast<const cuDoubleComplex*>(p); }
cuDoubleComplex* cz(zval* p) { return reinterpret_cast<cuDoubleComplex*>(p); }

// Cholesky in place (uplo), returns info (0 ok, >0 not positive definite)
int potrf(bse_ctx* ctx, zval* a, int k, cublasFillMode_t uplo, int* d_info) {
  size_t dws = 0, hws = 0;
  SOLVER_OK(cusolverDnXpotrf_bufferSize(ctx->solver, ctx->params, uplo, k, CUDA_C_64F, a, k, CUDA_C_64F, &dws, &hws));
  void* dbuf = solver_ws(ctx, dws);
  void* hbuf = host_ws(ctx, std::max<size_t>(hws, 16));
  SOLVER_OK(cusolverDnXpotrf(ctx->solver, ctx->params, uplo, k, CUDA_C_64F, a, k, CUDA_C_64F, dbuf, dws, hbuf, hws, d_info));
  int* info = reinterpret_cast<int*>(pinned(ctx, 1));
  CUDA_OK(cudaMemcpyAsync(info, d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return *info;
}

// hermitian eigendecomposition (values ascending in d_w; vectors overwrite a when want_vec)
void heevd(bse_ctx* ctx, zval* a, int k, double* d_w, bool want_vec, int* d_info) {
  const cusolverEigMode_t jobz = want_vec ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
  size_t dws = 0, hws = 0;
  SOLVER_OK(cusolverDnXsyevd_bufferSize(ctx->solver, ctx->params, jobz, CUBLAS_FILL_MODE_LOWER, k, CUDA_C_64F, a, k,
                                        CUDA_R_64F, d_w, CUDA_C_64F, &dws, &hws));
  void* dbuf = solver_ws(ctx, dws);
  void* hbuf = host_ws(ctx, std::max<size_t>(hws, 16));
  SOLVER_OK(cusolverDnXsyevd(ctx->solver, ctx->params, jobz, CUBLAS_FILL_MODE_LOWER, k, CUDA_C_64F, a, k, CUDA_R_64F,
                             d_w, CUDA_C_64F, dbuf, dws, hbuf, hws, d_info));
  int* info = reinterpret_cast<int*>(pinned(ctx, 1));
  CUDA_OK(cudaMemcpyAsync(info, d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  if (*info != 0) throw BseError(BSE_ENUMERICAL, "hermitian eigensolver failed (info " + std::to_string(*info) + ")");
}

void to_host(bse_ctx* ctx, double* h, const double* d, size_t count) {
  double* p = pinned(ctx, count);
  CUDA_OK(cudaMemcpyAsync(p, d, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  std::memcpy(h, p, count * sizeof(double));
}

void to_device(bse_ctx* ctx, double* d, const double* h, size_t count) {
  double* p = pinned(ctx, count);
  std::memcpy(p, h, count * sizeof(double));
  CUDA_OK(cudaMemcpyAsync(d, p, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
}

// max |G - I| of a k x k device matrix -> host
double defect_to_host(bse_ctx* ctx, const zval* g, int k, double* d_part) {
  const int nb = grid1d((int64_t)k * k, 256, 256);
  bse::defect_partial_kernel<<<nb, 256, 0, ctx->stream>>>(g, k, d_part);
  check_launch(ctx);
  bse::max_reduce_kernel<<<1, 32, 0, ctx->stream>>>(d_part, nb, d_part + nb);
  check_launch(ctx);
  double h = 0.0;
  to_host(ctx, &h, d_part + nb, 1);
  return h;
}

// ----------------------------------------------------------------------------
// CholQR (ortho.py:96-129), shifted CholQR3 fallback
// ----------------------------------------------------------------------------
// One CholQR pass on q (n x k) in place: G = Q^H Q (+ shift I), R = chol(G)
// (upper), Q <- Q R^{-1} with R^{-1} from a k x k TRSM and the product on the
// DMMA GEMM.  gram needs 2 k x k, tmp n x k.  Returns false when the Cholesky
// factorisation fails (ortho.py:113-119).
// One CholQR pass: G = Q^H Q (upper triangle only, hermitian by construction -- the reference's
// (G + G^H)/2, ortho.py:116-117, is then the identity on it), R = chol(G) upper, Q <- Q R^{-1}
// with the triangular R^{-1} (only the K rows <= column j contribute to column j).  gram holds
// 3 k x k blocks: [G -> R | R^{-1} | copy of G] (the copy feeds the folded defect check).
bool cholqr_pass(bse_ctx* ctx, zval* q, int64_t n, int64_t k, int64_t ldq, zval* gram, zval* tmp, zval* gws,
                 int* d_info, double shift, double* d_rdiag) {
  zgemm<bse::OPA_C>(ctx, k, k, n, 1.0, q, ldq, q, ldq, 0.0, gram, k, gws, bse::GEMM_UPPER);
  bse::herm_upper_kernel<<<grid1d(k * k), 256, 0, ctx->stream>>>(gram, (int)k);
  check_launch(ctx);
  if (shift != 0.0) {
    bse::add_diag_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(gram, (int)k, shift);
    check_launch(ctx);
  }
  CUDA_OK(cudaMemcpyAsync(gram + 2 * k * k, gram, (size_t)k * k * sizeof(zval), cudaMemcpyDeviceToDevice, ctx->stream));
  const int info = potrf(ctx, gram, (int)k, CUBLAS_FILL_MODE_UPPER, d_info);
  if (info != 0) return false;
  if (d_rdiag) {
    bse::absdiag_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(gram, (int)k, d_rdiag);
    check_launch(ctx);
  }
  zval* rinv = gram + k * k;
  bse::set_identity_kernel<<<grid1d(k * k), 256, 0, ctx->stream>>>(rinv, (int)k);
  check_launch(ctx);
  const cuDoubleComplex z1 = make_cuDoubleComplex(1.0, 0.0);
  BLAS_OK(cublasZtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)k,
                      (int)k, &z1, cz(gram), (int)k, cz(rinv), (int)k));
  CUDA_OK(cudaMemcpy2DAsync(tmp, sizeof(zval) * n, q, sizeof(zval) * ldq, sizeof(zval) * n, (size_t)k,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  zgemm<bse::OPA_N>(ctx, n, k, k, 1.0, tmp, n, rinv, k, 0.0, q, ldq, gws, bse::GEMM_B_UPPER);
  return true;
}

// Orthogonality defect max|Q^H Q - I| of the Q a CholQR pass produced, folded into that pass:
// Q^H Q = R^{-H} G R^{-1} with G the pass's own (exact) Gram (gram + 2 k^2) and R^{-1}
// (gram + k^2): two k x k x k products instead of a third n x k x k Gram (ortho.py:124).
double folded_defect(bse_ctx* ctx, zval* gram, int64_t k, zval* gws, double* dpart) {
  zval* rinv = gram + k * k;
  zval* g = gram + 2 * k * k;
  zval* x = gram;  // R is no longer needed
  zgemm<bse::OPA_N>(ctx, k, k, k, 1.0, g, k, rinv, k, 0.0, x, k, gws, bse::GEMM_B_UPPER);
  zgemm<bse::OPA_C>(ctx, k, k, k, 1.0, rinv, k, x, k, 0.0, g, k, gws);
  return defect_to_host(ctx, g, (int)k, dpart);
}

size_t cholqr_ws_bytes(int64_t n, int64_t k) {
  return al(3 * k * k * sizeof(zval)) + 2 * al(n * k * sizeof(zval)) +
         al(std::max({gemm_ws_bytes(k, k, n), gemm_ws_bytes(n, k, k), gemm_ws_bytes(k, k, k)}) + sizeof(zval)) +
         al(1024 * 8) + al(k * 8) + al(64) + 4096;
}

// ortho.py:96-129 on device.  Returns method (0 cholqr2, 1 shifted fallback);
// throws BSE_ERANK when no path yields a full-rank factor.
int cholqr_device(bse_ctx* ctx, zval* q, int64_t n, int64_t k, int64_t ldq, Scratch& sc) {
  if (k > n) throw BseError(BSE_ERANK, "cannot orthonormalize " + std::to_string(k) + " columns in dimension " +
                                           std::to_string(n));
  zval* gram = sc.take<zval>(3 * k * k);
  zval* tmp = sc.take<zval>(n * k);
  zval* gws = sc.take<zval>(std::max({gemm_ws_bytes(k, k, n), gemm_ws_bytes(n, k, k), gemm_ws_bytes(k, k, k)}) /
                                sizeof(zval) + 1);
  double* dpart = sc.take<double>(1024);
  double* rdiag = sc.take<double>(k);
  int* d_info = sc.take<int>(4);
  // keep the input for the fallback (ortho.py:126 restarts from x)
  bool ok = true;
  StepTimer tm(ctx, "cholqr");
  zval* x0 = sc.take<zval>(n * k);
  CUDA_OK(cudaMemcpy2DAsync(x0, sizeof(zval) * n, q, sizeof(zval) * ldq, sizeof(zval) * n, (size_t)k,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  for (int pass = 0; pass < 2 && ok; ++pass) {
    ok = cholqr_pass(ctx, q, n, k, ldq, gram, tmp, gws, d_info, 0.0, nullptr);
    tm.mark("cholqr pass", k);
  }
  if (ok) {
    const double defect = folded_defect(ctx, gram, k, gws, dpart);
    tm.mark("defect (folded into pass 2)", k);
    if (defect <= 1e-8) return 0;  // ortho.py:124-126 (NaN fails the test)
  }
  tm.mark("FALLBACK to shifted CholQR3", k);
  // Shifted CholeskyQR3 (Fukaya et al.): shift = 11 (n k + k (k + 1)) u ||X||_F^2, then CholQR2.
  CUDA_OK(cudaMemcpy2DAsync(q, sizeof(zval) * ldq, x0, sizeof(zval) * n, sizeof(zval) * n, (size_t)k,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  bse::frob2_kernel<<<(int)k, 256, 0, ctx->stream>>>(q, ldq, n, rdiag);
  check_launch(ctx);
  std::vector<double> f2(k);
  to_host(ctx, f2.data(), rdiag, k);
  double fro2 = 0.0;
  for (double v : f2) fro2 += v;
  const double u = std::ldexp(1.0, -53);
  const double shift = 11.0 * ((double)n * k + (double)k * (k + 1)) * u * fro2;
  // X = Q R3 R2 R1 with all three factors upper triangular, so |diag R(X)| is the
  // product of the per-pass diagonals; the rank test of ortho.py:86-93 runs on it.
  std::vector<double> dprod(k, 1.0), rd(k);
  auto pass_with_diag = [&](double sh) {
    if (!cholqr_pass(ctx, q, n, k, ldq, gram, tmp, gws, d_info, sh, rdiag)) return false;
    to_host(ctx, rd.data(), rdiag, k);
    for (int64_t i = 0; i < k; ++i) dprod[i] *= rd[i];
    return true;
  };
  if (!(fro2 > 0.0) || !pass_with_diag(shift))
    throw BseError(BSE_ERANK, "columns are numerically rank deficient (shifted Cholesky failed)");
  for (int pass = 0; pass < 2; ++pass)
    if (!pass_with_diag(0.0)) throw BseError(BSE_ERANK, "columns are numerically rank deficient (CholQR after shift failed)");
  const double dmax = *std::max_element(dprod.begin(), dprod.end()), dmin = *std::min_element(dprod.begin(), dprod.end());
  if (dmax == 0.0 || !(dmin > 1e-10 * dmax))
    throw BseError(BSE_ERANK, "columns are numerically rank deficient (diag ratio " + std::to_string(dmin) + " / " +
                                  std::to_string(dmax) + ")");
  zgemm<bse::OPA_C>(ctx, k, k, n, 1.0, q, ldq, q, ldq, 0.0, gram, k, gws);
  const double defect = defect_to_host(ctx, gram, (int)k, dpart);
  if (!(defect <= 1e-8)) throw BseError(BSE_ERANK, "orthonormalization failed (defect " + std::to_string(defect) + ")");
  return 1;
}

// Eigenvalues (no vectors) of the hermitian k x k `src`, computed on the context's second stream
// after the main stream reaches this point; the values and info land in pinned host memory.
// aux_eigvalsh_wait() joins and returns them.
void aux_eigvalsh_start(bse_ctx* ctx, const zval* src, zval* a, double* d_w, int* d_info, int k) {
  if (!ctx->aux) {
    CUDA_OK(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    SOLVER_OK(cusolverDnCreate(&ctx->aux_solver));
    SOLVER_OK(cusolverDnCreateParams(&ctx->aux_params));
    SOLVER_OK(cusolverDnSetStream(ctx->aux_solver, ctx->aux));
    for (cudaEvent_t& e : ctx->aux_ev) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  CUDA_OK(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
  CUDA_OK(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0));
  CUDA_OK(cudaMemcpyAsync(a, src, (size_t)k * k * sizeof(zval), cudaMemcpyDeviceToDevice, ctx->aux));
  size_t dws = 0, hws = 0;
  SOLVER_OK(cusolverDnXsyevd_bufferSize(ctx->aux_solver, ctx->aux_params, CUSOLVER_EIG_MODE_NOVECTOR,
                                        CUBLAS_FILL_MODE_LOWER, k, CUDA_C_64F, a, k, CUDA_R_64F, d_w, CUDA_C_64F, &dws,
                                        &hws));
  dws = std::max<size_t>(dws, 256);
  if (ctx->aux_dws_bytes < dws) {
    CUDA_OK(cudaStreamSynchronize(ctx->aux));
    if (ctx->aux_dws) CUDA_OK(cudaFree(ctx->aux_dws));
    CUDA_OK(cudaMalloc(&ctx->aux_dws, dws));
    ctx->aux_dws_bytes = dws;
  }
  if (ctx->aux_hws_bytes < std::max<size_t>(hws, 16)) {
    free(ctx->aux_hws);
    ctx->aux_hws = malloc(std::max<size_t>(hws, 16));
    ctx->aux_hws_bytes = std::max<size_t>(hws, 16);
  }
  if (ctx->aux_pinned_count < (size_t)k + 1) {
    if (ctx->aux_pinned) CUDA_OK(cudaFreeHost(ctx->aux_pinned));
    ctx->aux_pinned = nullptr;
    CUDA_OK(cudaMallocHost(&ctx->aux_pinned, (k + 1) * sizeof(double)));
    ctx->aux_pinned_count = k + 1;
  }
  SOLVER_OK(cusolverDnXsyevd(ctx->aux_solver, ctx->aux_params, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, k,
                             CUDA_C_64F, a, k, CUDA_R_64F, d_w, CUDA_C_64F, ctx->aux_dws, dws, ctx->aux_hws, hws,
                             d_info));
  CUDA_OK(cudaMemcpyAsync(ctx->aux_pinned, d_w, k * sizeof(double), cudaMemcpyDeviceToHost, ctx->aux));
  CUDA_OK(cudaMemcpyAsync(ctx->aux_pinned + k, d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->aux));
  CUDA_OK(cudaEventRecord(ctx->aux_ev[1], ctx->aux));
}

void aux_eigvalsh_wait(bse_ctx* ctx, std::vector<double>& w, int k) {
  CUDA_OK(cudaEventSynchronize(ctx->aux_ev[1]));
  CUDA_OK(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));  // scratch reuse stays ordered
  int info = 0;
  std::memcpy(&info, ctx->aux_pinned + k, sizeof(int));
  if (info != 0) throw BseError(BSE_ENUMERICAL, "hermitian eigensolver failed (info " + std::to_string(info) + ")");
  w.assign(ctx->aux_pinned, ctx->aux_pinned + k);
}

// copy one k x k factor into slot `slot` of the registered capture buffer (no-op when none)
void capture_kk(bse_ctx* ctx, int slot, const zval* src, int64_t k) {
  if (!ctx->rr_capture) return;
  CUDA_OK(cudaMemcpyAsync(ctx->rr_capture + (size_t)slot * k * k, src, (size_t)k * k * sizeof(zval),
                          cudaMemcpyDeviceToDevice, ctx->stream));
}

size_t pencil_ws_bytes(int64_t k) { return 3 * al((size_t)k * k * sizeof(zval)) + 2 * al(k * 8) + al(k * 4) + al(64); }

// Small hermitian pencil of the oblique RR (rayleigh_ritz.py:113-137) on k x k device data:
// w = Q^H S H Q and g2 = Q2^H Q2 (raw sums, overwritten).  Returns ascending Ritz values on the
// host and the sorted back-transform wvec = L^{-H} y[:, order] on the device.
// mode 0: the whole pencil (rayleigh_ritz.py:113-137); mode 1: only |lambda|_min(M) into
// *h_lam_min_m (no check); mode 2: the pencil without the eigenvalues of M (the caller has them)
void rr_pencil(bse_ctx* ctx, zval* w, zval* g2, int64_t k, double* h_lam, zval* wvec, double* h_lam_min_m,
               Scratch& sc, int mode = 0) {
  const size_t kk = (size_t)k * k;
  StepTimer tm(ctx, "rr_pencil");
  zval* mm = sc.take<zval>(kk);
  zval* tmp = sc.take<zval>(kk);
  zval* g = sc.take<zval>(kk);
  double* d_w = sc.take<double>(k);
  int* d_perm = sc.take<int>(k);
  int* d_info = sc.take<int>(4);
  // W and Q2^H Q2 are hermitian: their upper triangles (GEMM_UPPER) define them
  bse::herm_upper_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(w, (int)k);
  check_launch(ctx);
  bse::form_m_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(g2, mm, (int)k);
  check_launch(ctx);
  bse::herm_upper_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(mm, (int)k);
  check_launch(ctx);
  capture_kk(ctx, 0, w, k);
  capture_kk(ctx, 2, mm, k);
  std::vector<double> hw(k);
  // :116-120  |lambda|_min(M) >= 1e-8 -- the eigenvalues of M run on the second stream while this
  // one factors W and solves G; the checks below keep the reference's order (M first, then the
  // Cholesky of W, then theta ~ 0), so the same error is raised for the same input
  bool m_pending = false;
  auto check_m = [&]() {
    if (!m_pending) return;
    m_pending = false;
    std::vector<double> wm;
    aux_eigvalsh_wait(ctx, wm, (int)k);
    double lmm = INFINITY;
    for (double v : wm) lmm = std::min(lmm, std::fabs(v));
    if (h_lam_min_m) *h_lam_min_m = lmm;
    tm.mark("eigvalsh(M) joined", k);
    if (mode == 1) return;
    if (!(lmm >= 1e-8))
      throw BseError(BSE_EHERMITIAN_RQ, "|lambda_min(Q*SQ)| = " + std::to_string(lmm) + " below 1e-8");
  };
  if (mode != 2) {
    int* m_info = d_info + 1;
    aux_eigvalsh_start(ctx, mm, tmp, d_w + 0, m_info, (int)k);
    m_pending = true;
    if (mode == 1) {
      check_m();
      return;
    }
  }
  double* d_wg = sc.take<double>(k);  // eigenvalues of G (d_w belongs to the second stream)
  // :121-126  L = chol(W)
  if (potrf(ctx, w, (int)k, CUBLAS_FILL_MODE_LOWER, d_info) != 0) {
    check_m();
    throw BseError(BSE_EHERMITIAN_RQ, "Cholesky of Q*SHQ failed; S*H is not definite on the subspace");
  }
  capture_kk(ctx, 1, w, k);  // L in the lower triangle (the caller drops the upper)
  // :127-129  G = L^{-1} M L^{-H}, hermitised
  const cuDoubleComplex z1 = make_cuDoubleComplex(1.0, 0.0);
  CUDA_OK(cudaMemcpyAsync(g, mm, kk * sizeof(zval), cudaMemcpyDeviceToDevice, ctx->stream));
  BLAS_OK(cublasZtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)k,
                      (int)k, &z1, cz(w), (int)k, cz(g), (int)k));
  BLAS_OK(cublasZtrsm(ctx->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, (int)k,
                      (int)k, &z1, cz(w), (int)k, cz(g), (int)k));
  bse::hermitize_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(g, (int)k);
  check_launch(ctx);
  capture_kk(ctx, 3, g, k);
  tm.mark("chol(W), G = L^-1 M L^-H", k);
  // :130-133  theta, y = eigh(G); lambda = 1/theta
  heevd(ctx, g, (int)k, d_wg, true, d_info);
  to_host(ctx, hw.data(), d_wg, k);
  tm.mark("eigh(G)", k);
  check_m();
  double tmin = INFINITY;
  for (double v : hw) tmin = std::min(tmin, std::fabs(v));
  if (tmin < 2.220446049250313e-16) throw BseError(BSE_EHERMITIAN_RQ, "reduced spectrum touches zero; cannot invert");
  std::vector<double> lam(k);
  for (int64_t i = 0; i < k; ++i) lam[i] = 1.0 / hw[i];
  std::vector<int> order(k);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lam[a] < lam[b]; });
  for (int64_t i = 0; i < k; ++i) h_lam[i] = lam[order[i]];
  // :134  w = L^{-H} y, columns in ascending-lambda order
  BLAS_OK(cublasZtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, (int)k,
                      (int)k, &z1, cz(w), (int)k, cz(g), (int)k));
  {
    std::vector<double> packed((k + 1) / 2 + 1);
    std::memcpy(packed.data(), order.data(), sizeof(int) * k);
    to_device(ctx, reinterpret_cast<double*>(d_perm), packed.data(), (k + 1) / 2);
  }
  bse::gather_cols_kernel<<<dim3(1, (unsigned)k), 256, 0, ctx->stream>>>(g, k, wvec, k, k, d_perm);
  check_launch(ctx);
}

// ---------------------------------------------------------------------------------------------
// complex64 filter on tcgen05 (c64.cuh): TMA tensor maps and the step driver
// ---------------------------------------------------------------------------------------------
// 3-D fp32 tensor map with a 64-byte-swizzled box (b0 x b1 x b2), strides in bytes
CUtensorMap map3d(const float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2, uint32_t b0,
                  uint32_t b1, uint32_t b2) {
  CUtensorMap map;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw BseError(BSE_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return map;
}

inline int64_t pad4(int64_t m) { return (m + 3) & ~int64_t(3); }

// P planes: 4 x [mo rows][2 mpi] fp32 (mpi = pad4(kc));  view (j < kc, row i < mo, part)
void c64_p_maps(bse::c64::Maps& mp_, const float* pplanes, int64_t mo, int64_t kc) {
  const int64_t mpi = pad4(kc), plane = mo * 2 * mpi;
  for (int q = 0; q < 4; ++q)
    mp_.p[q] = map3d(pplanes + q * plane, kc, mo, 2, 2 * mpi * 4, mpi * 4, bse::c64::BKE, bse::c64::BM, 1);
}

// X planes of one block: 8 x [k cols][2 mpi] fp32;  view (j < kc, half, col); rows >= kc zero-filled
void c64_x_maps(bse::c64::Maps& mp_, const float* const planes[8], int64_t kc, int64_t k) {
  const int64_t mpi = pad4(kc);
  for (int q = 0; q < 8; ++q)
    mp_.x[q] = map3d(planes[q], kc, 2, k, mpi * 4, 2 * mpi * 4, bse::c64::BKE, 1, bse::c64::BN);
}

struct C64Step {
  int64_t mo, kc, k;
  const float* x[8];     // input planes (input layout)
  const float* prev[4];  // y_prev planes (output layout), null: beta = 0
  float* out[8];         // output planes, or raw (out[0] = Re, out[1] = Im)
  double alpha, beta, shift;
  int64_t shift_lo, shift_hi, s_off;
  bool raw;
};

// CTA-pair (cta_group::2) variant of the c64 step for wide blocks: 13% faster at k = 1200, 5-7%
// slower at k = 300-600 (profiles/r01/c64_pair_vs_single.txt).  BSE200_C64_PAIR=0 / 1 forces it.
bool c64_pair(int64_t k) {
  const char* v = std::getenv("BSE200_C64_PAIR");
  return v && v[0] ? v[0] != '0' : k >= 900;
}

void c64_step(bse_ctx* ctx, bse::c64::Maps& maps, const C64Step& st) {
  ensure_smem(ctx, (const void*)bse::c64::step_kernel<false>, (int)bse::c64::SMEM);
  ensure_smem(ctx, (const void*)bse::c64::step_kernel<true>, (int)bse::c64::PAIR_SMEM);
  c64_x_maps(maps, st.x, st.kc, st.k);
  bse::c64::StepArgs a{};
  a.mo = (int)st.mo;
  a.mpo = (int)pad4(st.mo);
  a.kc = (int)st.kc;
  a.mpi = (int)pad4(st.kc);
  a.k = (int)st.k;
  a.skip_b = (ctx->ham_flags & BSE_HAM_B_ZERO) ? 1 : 0;
  for (int q = 0; q < 4; ++q) {
    a.x[q] = st.x[q];
    a.p[q] = st.prev[q];
  }
  for (int q = 0; q < 8; ++q) a.out[q] = st.out[q];
  a.alpha = (float)st.alpha;
  a.beta = st.prev[0] ? (float)st.beta : 0.f;
  a.shift = (float)st.shift;
  a.shift_lo = (int)st.shift_lo;
  a.shift_hi = (int)st.shift_hi;
  a.s_off = (int)st.s_off;
  a.raw = st.raw ? 1 : 0;
  const unsigned nt = (unsigned)((st.k + bse::c64::BN - 1) / bse::c64::BN);
  const unsigned mt = (unsigned)((st.mo + bse::c64::BM - 1) / bse::c64::BM);
  if (c64_pair(st.k)) {
    // CTA pairs (clusters along x) over adjacent row tiles, column tiles fastest (c64.cuh; an odd
    // row-tile count gets one all-padding CTA)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * nt, (mt + 1) / 2);
    cfg.blockDim = dim3(bse::c64::THREADS);
    cfg.dynamicSmemBytes = bse::c64::PAIR_SMEM;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_OK(cudaLaunchKernelEx(&cfg, bse::c64::step_kernel<true>, maps, a));
  } else {
    bse::c64::step_kernel<false><<<dim3(nt, mt), bse::c64::THREADS, bse::c64::SMEM, ctx->stream>>>(maps, a);
  }
  check_launch(ctx);
}

// the 8 planes of a plane set: consecutive blocks of 2 pad4(rows) k floats
void plane_set(float* base, int64_t rows, int64_t k, float* (&q)[8]) {
  const int64_t blk = 2 * pad4(rows) * k;
  for (int i = 0; i < 8; ++i) q[i] = base + i * blk;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* bse_version(void) { return "bse200 0.1 (sm_100a, FP64 DMMA)"; }

int bse_ctx_create(int device, bse_ctx** out) {
  if (!out) return BSE_EVALIDATION;
  *out = nullptr;
  bse_ctx* ctx = new bse_ctx();
  ctx->device = device;
  if (const char* g = std::getenv("BSE200_RS_GROUP_ROWS")) ctx->rs_group_rows = std::max(0, std::atoi(g));
  if (const char* g = std::getenv("BSE200_RS_KSPLIT")) ctx->rs_ksplit = std::max(0, std::min(4, std::atoi(g)));
  try {
    CUDA_OK(cudaSetDevice(device));
    BLAS_OK(cublasCreate(&ctx->blas));
    SOLVER_OK(cusolverDnCreate(&ctx->solver));
    SOLVER_OK(cusolverDnCreateParams(&ctx->params));
  } catch (const BseError& e) {
    delete ctx;
    return e.code;
  }
  *out = ctx;
  return BSE_OK;
}

void bse_ctx_destroy(bse_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->sws) cudaFree(ctx->sws);
  if (ctx->gv) cudaFree(ctx->gv);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  free(ctx->hws);
  if (ctx->aux) {
    cudaStreamSynchronize(ctx->aux);
    if (ctx->aux_dws) cudaFree(ctx->aux_dws);
    if (ctx->aux_pinned) cudaFreeHost(ctx->aux_pinned);
    free(ctx->aux_hws);
    for (cudaEvent_t e : ctx->aux_ev)
      if (e) cudaEventDestroy(e);
    if (ctx->aux_params) cusolverDnDestroyParams(ctx->aux_params);
    if (ctx->aux_solver) cusolverDnDestroy(ctx->aux_solver);
    cudaStreamDestroy(ctx->aux);
  }
  if (ctx->params) cusolverDnDestroyParams(ctx->params);
  if (ctx->solver) cusolverDnDestroy(ctx->solver);
  if (ctx->blas) cublasDestroy(ctx->blas);
  delete ctx;
}

int bse_set_hamiltonian_flags(bse_ctx* ctx, unsigned flags) {
  return guarded(ctx, [&] { ctx->ham_flags = flags; });
}

int bse_set_filter_algorithm(bse_ctx* ctx, int complex_mults) {
  return guarded(ctx, [&] {
    if (!filter_code_valid(complex_mults))
      throw BseError(BSE_EVALIDATION, "filter algorithm must be 4, 82, 86, 88, 90, 92, 94, 96, 97 or 98 (include/bse200.h)");
    ctx->filter_cm = complex_mults;
  });
}

int bse_set_stream(bse_ctx* ctx, void* stream) {
  return guarded(ctx, [&] {
    ctx->stream = static_cast<cudaStream_t>(stream);
    BLAS_OK(cublasSetStream(ctx->blas, ctx->stream));
    SOLVER_OK(cusolverDnSetStream(ctx->solver, ctx->stream));
  });
}

const char* bse_last_error(const bse_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int64_t bse_launch_count(const bse_ctx* ctx) { return ctx ? ctx->launches : 0; }

int bse_apply_h(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_x, int64_t ldx,
                void* d_y, int64_t ldy, int64_t k, double low_sign) {
  return guarded(ctx, [&] {
    if (m < 0 || k < 0 || lda < m || ldx < 2 * m || ldy < 2 * m) throw BseError(BSE_EVALIDATION, "bad shapes");
    apply_h(ctx, d_ab, lda, m, static_cast<const zval*>(d_x), ldx, static_cast<zval*>(d_y), ldy, k, low_sign, d_sd);
  });
}

int bse_filter_step(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_y,
                    const void* d_yprev, void* d_ynext, int64_t ld, int64_t k, double c, double alpha, double beta) {
  return guarded(ctx, [&] {
    if (m < 0 || k < 0 || lda < m || ld < 2 * m) throw BseError(BSE_EVALIDATION, "bad shapes");
    if (k == 0 || m == 0) return;
    filter_step(ctx, d_ab, d_sd, lda, m, static_cast<const zval*>(d_y), static_cast<const zval*>(d_yprev),
                static_cast<zval*>(d_ynext), ld, k, c, alpha, beta);
  });
}

int bse_make_sum_planes(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, int64_t cols, void* d_sd) {
  return guarded(ctx, [&] {
    if (m <= 0 || cols <= 0) return;
    bse::sum_planes_kernel<<<grid1d(m * cols, 256, 148 * 32), 256, 0, ctx->stream>>>(static_cast<const zval*>(d_ab), lda,
                                                                                   m, cols, static_cast<zval*>(d_sd));
    check_launch(ctx);
  });
}

int bse_chebyshev_filter(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, void* d_v,
                         int64_t ld, int64_t k, int deg, double c, double e, double s, void* d_work) {
  return guarded(ctx, [&] {
    if (deg < 2 || deg % 2) throw BseError(BSE_EVALIDATION, "filter degree must be even and >= 2");
    if (!(e > 0)) throw BseError(BSE_EVALIDATION, "filter half width must be positive");
    if (m < 0 || k < 0 || lda < m || ld < 2 * m) throw BseError(BSE_EVALIDATION, "bad shapes");
    if (k == 0 || m == 0) return;
    // chebyshev.py:58-74 with three rotating buffers {v, w0, w1}
    zval* bufs[3] = {static_cast<zval*>(d_v), static_cast<zval*>(d_work), static_cast<zval*>(d_work) + ld * k};
    const double sigma1 = e / (s - c);
    double sigma = sigma1;
    int prev = 0, cur = 1;
    filter_step(ctx, d_ab, d_sd, lda, m, bufs[0], nullptr, bufs[1], ld, k, c, sigma1 / e, 0.0);
    for (int step = 2; step <= deg; ++step) {
      const double sigma_new = 1.0 / (2.0 / sigma1 - sigma);
      const int nxt = 3 - prev - cur;
      // y_next = (2 s'/e)(H y - c y) - (s s') y_prev ; written over the free buffer
      filter_step(ctx, d_ab, d_sd, lda, m, bufs[cur], bufs[prev], bufs[nxt], ld, k, c, 2.0 * sigma_new / e,
                  sigma * sigma_new);
      prev = cur;
      cur = nxt;
      sigma = sigma_new;
    }
    if (cur != 0)
      CUDA_OK(cudaMemcpyAsync(bufs[0], bufs[cur], sizeof(zval) * ld * k, cudaMemcpyDeviceToDevice, ctx->stream));
  });
}

int bse_make_rs_planes(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t mr, int64_t kc, void* d_g, int64_t ldg) {
  return guarded(ctx, [&] {
    if (mr < 0 || kc < 0 || lda < mr || ldg < mr || (ldg & 1))
      throw BseError(BSE_EVALIDATION, "bad shapes (ldg must be even, >= mr)");
    if (mr == 0 || kc == 0) return;
    bse::rs_planes_kernel<<<grid1d(mr * kc, 256, 148 * 32), 256, 0, ctx->stream>>>(
        static_cast<const zval*>(d_ab), lda, mr, kc, static_cast<double*>(d_g), ldg);
    check_launch(ctx);
  });
}

int bse_set_rr_capture(bse_ctx* ctx, void* d_buf) {
  return guarded(ctx, [&] { ctx->rr_capture = static_cast<zval*>(d_buf); });
}

int bse_set_rs_planes(bse_ctx* ctx, const void* d_ab, int64_t m, const void* d_g, int64_t ldg) {
  return guarded(ctx, [&] {
    if (d_g && (m <= 0 || ldg < m || (ldg & 1))) throw BseError(BSE_EVALIDATION, "bad shapes (ldg must be even, >= m)");
    ctx->rs_ab = d_g ? d_ab : nullptr;
    ctx->rs_g = static_cast<const double*>(d_g);
    ctx->rs_ldg = d_g ? ldg : 0;
    ctx->rs_m = d_g ? m : 0;
  });
}

int bse_chebyshev_filter_rs(bse_ctx* ctx, const void* d_g, int64_t ldg, int64_t m, void* d_v, int64_t ld, int64_t k,
                            int deg, double c, double e, double s, void* d_work) {
  return guarded(ctx, [&] {
    if (deg < 2 || deg % 2) throw BseError(BSE_EVALIDATION, "filter degree must be even and >= 2");
    if (!(e > 0)) throw BseError(BSE_EVALIDATION, "filter half width must be positive");
    if (m < 0 || k < 0 || ldg < m || (ldg & 1) || ld < 2 * m) throw BseError(BSE_EVALIDATION, "bad shapes");
    if (ctx->ham_flags & BSE_HAM_B_ZERO) throw BseError(BSE_EVALIDATION, "the real-split filter needs B != 0");
    if (k == 0 || m == 0) return;
    const double* g = static_cast<const double*>(d_g);
    zval* bufs[3] = {static_cast<zval*>(d_v), static_cast<zval*>(d_work), static_cast<zval*>(d_work) + ld * k};
    const int fb = grid1d(m * k, 256, 148 * 16);
    bse::rs_fold_kernel<<<fb, 256, 0, ctx->stream>>>(bufs[0], bufs[0], ld, ld, m, k, 1.0, 1.0);
    check_launch(ctx);
    // the recurrence of bse_chebyshev_filter (chebyshev.py:58-74) in the folded basis
    const double sigma1 = e / (s - c);
    double sigma = sigma1;
    int prev = 0, cur = 1;
    rs_step(ctx, g, ldg, m, bufs[0], nullptr, bufs[1], ld, k, c, sigma1 / e, 0.0);
    for (int step = 2; step <= deg; ++step) {
      const double sigma_new = 1.0 / (2.0 / sigma1 - sigma);
      const int nxt = 3 - prev - cur;
      rs_step(ctx, g, ldg, m, bufs[cur], bufs[prev], bufs[nxt], ld, k, c, 2.0 * sigma_new / e, sigma * sigma_new);
      prev = cur;
      cur = nxt;
      sigma = sigma_new;
    }
    // unfold into d_v: X1 = (x + y) / 2, X2 = (x - y) / 2
    bse::rs_fold_kernel<<<fb, 256, 0, ctx->stream>>>(bufs[cur], bufs[0], ld, ld, m, k, 0.5, 0.5);
    check_launch(ctx);
  });
}

int bse_residuals(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, const void* d_v, int64_t ldv, int64_t k,
                  const double* h_lam, double* h_res) {
  return guarded(ctx, [&] {
    if (k == 0) return;
    Scratch sc(ctx, al(k * 8) * 2 + al(resid_part_count(m, k) * 8));
    double* d_lam = sc.take<double>(k);
    double* d_out = sc.take<double>(k);
    double* d_part = sc.take<double>(resid_part_count(m, k));
    to_device(ctx, d_lam, h_lam, k);
    residual_norms(ctx, d_ab, lda, m, static_cast<const zval*>(d_v), ldv, k, d_lam, d_part, d_out);
    to_host(ctx, h_res, d_out, k);
  });
}

int bse_zgemm_cn(bse_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const void* d_a, int64_t lda,
                 const void* d_b, int64_t ldb, double beta, void* d_c, int64_t ldc) {
  return guarded(ctx, [&] {
    Scratch sc(ctx, gemm_ws_bytes(M, N, K));
    zval* ws = gemm_ws_bytes(M, N, K) ? sc.take<zval>((size_t)splitk_for(M, N, K) * M * N) : nullptr;
    zgemm<bse::OPA_C>(ctx, M, N, K, alpha, static_cast<const zval*>(d_a), lda, static_cast<const zval*>(d_b), ldb,
                      beta, static_cast<zval*>(d_c), ldc, ws);
  });
}

int bse_zgemm_nn(bse_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const void* d_a, int64_t lda,
                 const void* d_b, int64_t ldb, double beta, void* d_c, int64_t ldc) {
  return guarded(ctx, [&] {
    Scratch sc(ctx, gemm_ws_bytes(M, N, K));
    zval* ws = gemm_ws_bytes(M, N, K) ? sc.take<zval>((size_t)splitk_for(M, N, K) * M * N) : nullptr;
    zgemm<bse::OPA_N>(ctx, M, N, K, alpha, static_cast<const zval*>(d_a), lda, static_cast<const zval*>(d_b), ldb,
                      beta, static_cast<zval*>(d_c), ldc, ws);
  });
}

int bse_cholqr(bse_ctx* ctx, void* d_q, int64_t n, int64_t k, int64_t ldq, int* h_method) {
  return guarded(ctx, [&] {
    if (k == 0) {
      if (h_method) *h_method = 0;
      return;
    }
    Scratch sc(ctx, cholqr_ws_bytes(n, k));
    zval* q = static_cast<zval*>(d_q);
    const int method = cholqr_device(ctx, q, n, k, ldq, sc);
    bse::phase_fix_kernel<<<(int)k, 256, 0, ctx->stream>>>(q, ldq, n);
    check_launch(ctx);
    if (h_method) *h_method = method;
  });
}

int bse_fix_phases(bse_ctx* ctx, void* d_q, int64_t n, int64_t k, int64_t ldq) {
  return guarded(ctx, [&] {
    if (k == 0 || n == 0) return;
    bse::phase_fix_kernel<<<(int)k, 256, 0, ctx->stream>>>(static_cast<zval*>(d_q), ldq, n);
    check_launch(ctx);
  });
}

int bse_s_orthonormalize(bse_ctx* ctx, void* d_v, int64_t n, int64_t k, int64_t ldv, const void* d_ylocked,
                         int64_t l, int64_t ldy, int* h_method) {
  return guarded(ctx, [&] {
    if (n % 2) throw BseError(BSE_EVALIDATION, "S needs an even row count");
    if (k == 0) {
      if (h_method) *h_method = 0;
      return;
    }
    zval* v = static_cast<zval*>(d_v);
    const int64_t m = n / 2;
    size_t need = cholqr_ws_bytes(n, std::max(k, l));
    if (l > 0) need += al(n * l * sizeof(zval)) + al(l * k * sizeof(zval)) + gemm_ws_bytes(l, k, n) + gemm_ws_bytes(n, k, l);
    Scratch sc(ctx, need);
    if (l > 0) {
      // ortho.py:148-155: orthonormal basis of span(S Y_locked), then v -= basis (basis^H v)
      zval* basis = sc.take<zval>(n * l);
      zval* proj = sc.take<zval>(l * k);
      zval* gws = sc.take<zval>(std::max(gemm_ws_bytes(l, k, n), gemm_ws_bytes(n, k, l)) / sizeof(zval) + 1);
      bse::sflip_copy_kernel<<<grid1d(n * l), 256, 0, ctx->stream>>>(static_cast<const zval*>(d_ylocked), ldy, basis,
                                                                       n, m, l);
      check_launch(ctx);
      {
        Scratch inner = sc;  // carve the basis CholQR scratch after ours
        cholqr_device(ctx, basis, n, l, n, inner);
      }
      zgemm<bse::OPA_C>(ctx, l, k, n, 1.0, basis, n, v, ldv, 0.0, proj, l, gws);
      zgemm<bse::OPA_N>(ctx, n, k, l, -1.0, basis, n, proj, l, 1.0, v, ldv, gws);
    }
    Scratch rest = sc;
    const int method = cholqr_device(ctx, v, n, k, ldv, rest);
    bse::phase_fix_kernel<<<(int)k, 256, 0, ctx->stream>>>(v, ldv, n);
    check_launch(ctx);
    if (h_method) *h_method = method;
  });
}

// Incrementally maintained orthonormal basis of span(S Y_locked) (SURVEY.md §7 "Locked basis"): the
// reference re-runs a Householder QR of the whole n x l flipped locked block every iteration
// (ortho.py:149-150); the span only grows by the newly locked columns, so they alone are
// S-flipped, projected twice against the existing basis (block classical Gram-Schmidt, BCGS2) and
// CholQR'd.  Same span, hence the same projector, to rounding.
int bse_extend_sbasis(bse_ctx* ctx, void* d_basis, int64_t n, int64_t ldb, int64_t l_old, const void* d_ynew,
                      int64_t ldy, int64_t c) {
  return guarded(ctx, [&] {
    if (n % 2) throw BseError(BSE_EVALIDATION, "S needs an even row count");
    if (c <= 0) return;
    if (ldb < n || ldy < n || l_old < 0) throw BseError(BSE_EVALIDATION, "bad shapes");
    zval* basis = static_cast<zval*>(d_basis);
    zval* bn = basis + l_old * ldb;
    const int64_t m = n / 2;
    size_t need = cholqr_ws_bytes(n, c);
    if (l_old > 0) need += al(l_old * c * sizeof(zval)) + std::max(gemm_ws_bytes(l_old, c, n), gemm_ws_bytes(n, c, l_old)) + 256;
    Scratch sc(ctx, need);
    bse::sflip_copy_kernel<<<grid1d(n * c), 256, 0, ctx->stream>>>(static_cast<const zval*>(d_ynew), ldy, bn, ldb, m,
                                                                     c);
    check_launch(ctx);
    if (l_old > 0) {
      zval* proj = sc.take<zval>(l_old * c);
      zval* gws = sc.take<zval>(std::max(gemm_ws_bytes(l_old, c, n), gemm_ws_bytes(n, c, l_old)) / sizeof(zval) + 1);
      for (int pass = 0; pass < 2; ++pass) {
        zgemm<bse::OPA_C>(ctx, l_old, c, n, 1.0, basis, ldb, bn, ldb, 0.0, proj, l_old, gws);
        zgemm<bse::OPA_N>(ctx, n, c, l_old, -1.0, basis, ldb, proj, l_old, 1.0, bn, ldb, gws);
      }
    }
    Scratch rest = sc;
    cholqr_device(ctx, bn, n, c, ldb, rest);
  });
}

// ortho.py:132-158 with the locked space given by its orthonormal basis (bse_extend_sbasis):
// v <- v - basis (basis^H v), CholQR2 (+ shifted fallback), phase convention.
int bse_s_orthonormalize_basis(bse_ctx* ctx, void* d_v, int64_t n, int64_t k, int64_t ldv, const void* d_basis,
                               int64_t l, int64_t ldb, int* h_method) {
  return guarded(ctx, [&] {
    if (k == 0) {
      if (h_method) *h_method = 0;
      return;
    }
    zval* v = static_cast<zval*>(d_v);
    const zval* basis = static_cast<const zval*>(d_basis);
    size_t need = cholqr_ws_bytes(n, k);
    if (l > 0) need += al(l * k * sizeof(zval)) + std::max(gemm_ws_bytes(l, k, n), gemm_ws_bytes(n, k, l)) + 256;
    Scratch sc(ctx, need);
    if (l > 0) {
      zval* proj = sc.take<zval>(l * k);
      zval* gws = sc.take<zval>(std::max(gemm_ws_bytes(l, k, n), gemm_ws_bytes(n, k, l)) / sizeof(zval) + 1);
      zgemm<bse::OPA_C>(ctx, l, k, n, 1.0, basis, ldb, v, ldv, 0.0, proj, l, gws);
      zgemm<bse::OPA_N>(ctx, n, k, l, -1.0, basis, ldb, proj, l, 1.0, v, ldv, gws);
    }
    Scratch rest = sc;
    const int method = cholqr_device(ctx, v, n, k, ldv, rest);
    bse::phase_fix_kernel<<<(int)k, 256, 0, ctx->stream>>>(v, ldv, n);
    check_launch(ctx);
    if (h_method) *h_method = method;
  });
}

int bse_rr_hermitian(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_q,
                     int64_t ldq, int64_t k, double* h_lam, void* d_vout, int64_t ldvout, double* h_lam_min_m,
                     double* h_res) {
  return guarded(ctx, [&] {
    if (k == 0) return;
    if (!d_ab && !rs_active(ctx, d_ab, m))
      throw BseError(BSE_EVALIDATION, "null operator: a planes-only operator needs bse_set_rs_planes(ctx, NULL, m, g, ldg)");
    const int64_t n = 2 * m;
    const zval* q = static_cast<const zval*>(d_q);
    zval* vout = static_cast<zval*>(d_vout);
    const size_t kk = (size_t)k * k;
    const size_t gwsb = std::max({gemm_ws_bytes(k, k, n), gemm_ws_bytes(k, k, m), gemm_ws_bytes(n, k, k)});
    const bool rs = (k > 1 || !d_ab) && rs_active(ctx, d_ab, m);
    Scratch sc(ctx, (h_res ? 2 : 1) * al(n * k * sizeof(zval)) + 3 * al(kk * sizeof(zval)) + 4 * al(k * 8) + gwsb +
                        pencil_ws_bytes(k) + 4096 + (rs ? al(n * k * sizeof(zval)) : 0));
    zval* t = sc.take<zval>(n * k);
    zval* fold = rs ? sc.take<zval>(n * k) : nullptr;
    zval* u = h_res ? sc.take<zval>(n * k) : nullptr;
    double* d_lam = sc.take<double>(k);
    double* d_rinv = sc.take<double>(k);
    double* d_r2 = sc.take<double>(k);
    zval* w = sc.take<zval>(kk);
    zval* g2 = sc.take<zval>(kk);
    zval* wvec = sc.take<zval>(kk);
    double* d_norm = sc.take<double>(k);
    zval* gws = sc.take<zval>(gwsb / sizeof(zval) + 1);
    StepTimer tm(ctx, "rr_hermitian");
    // rayleigh_ritz.py:112-115: T = S H Q ; W = Q^H T ; Q2^H Q2
    apply_h(ctx, d_ab, lda, m, q, ldq, t, n, k, -1.0, d_sd, fold);
    tm.mark("T = S H Q", k);
    zgemm<bse::OPA_C>(ctx, k, k, n, 1.0, q, ldq, t, n, 0.0, w, k, gws, bse::GEMM_UPPER);
    zgemm<bse::OPA_C>(ctx, k, k, m, 1.0, q + m, ldq, q + m, ldq, 0.0, g2, k, gws, bse::GEMM_UPPER);
    tm.mark("grams W, Q2^H Q2 (upper triangles)", k);
    Scratch rest = sc;
    rr_pencil(ctx, w, g2, k, h_lam, wvec, h_lam_min_m, rest);
    tm.mark("pencil", k);
    // :135-136  V = Q w (sorted) ; unit columns
    zgemm<bse::OPA_N>(ctx, n, k, k, 1.0, q, ldq, wvec, k, 0.0, vout, ldvout, gws);
    bse::colnorm_kernel<<<(int)k, 256, 0, ctx->stream>>>(vout, ldvout, n, d_norm);
    check_launch(ctx);
    bse::colscale_inv_kernel<<<dim3(grid1d(n, 256, 64), (unsigned)k), 256, 0, ctx->stream>>>(vout, ldvout, n, d_norm);
    check_launch(ctx);
    tm.mark("V = Q w, normalise", k);
    if (h_res) {
      // residuals from the RR intermediate: H V = S T w / |Q w| (saves the H application of
      // rayleigh_ritz.py:188; 8 n k^2 instead of 8 n^2 k)
      zgemm<bse::OPA_N>(ctx, n, k, k, 1.0, t, n, wvec, k, 0.0, u, n, gws);
      to_device(ctx, d_lam, h_lam, k);
      bse::recip_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(d_norm, d_rinv, (int)k);
      check_launch(ctx);
      bse::resid_from_rr_kernel<<<(int)k, 256, 0, ctx->stream>>>(u, n, vout, ldvout, n, m, d_rinv, d_lam, d_r2);
      check_launch(ctx);
      to_host(ctx, h_res, d_r2, k);
      for (int64_t i = 0; i < k; ++i) h_res[i] = std::sqrt(h_res[i]);
      tm.mark("residuals from S T w", k);
    }
  });
}

size_t backup_ws_bytes(int64_t k) {
  const size_t kk = (size_t)k * k;
  return 5 * al(kk * sizeof(zval)) + 2 * al(k * 16) + 2 * al(k * 8) + al(k * 4) + al(64) + gemm_ws_bytes(k, k, k) +
         4096;
}

// k x k tail of the backup projection (rayleigh_ritz.py:160-175) from summed partials:
// g = Q^H S H Q (overwritten), w = Q^H H Q, g2 = Q2^H Q2 (overwritten).  Ascending real parts of
// eig(g') with g' = diag(d)^{-1} (g - offdiag(M) w), M = I - 2 g2; y = the sorted eigenvectors.
void backup_pencil(bse_ctx* ctx, zval* g, const zval* w, zval* g2, int64_t k, double* h_lam, zval* yperm,
                   double* h_lam_min_m, Scratch& sc) {
  const size_t kk = (size_t)k * k;
  zval* mm = sc.take<zval>(kk);
  zval* tmp = sc.take<zval>(kk);
  zval* y = sc.take<zval>(kk);
  zval* d_ev = sc.take<zval>(k);
  double* d_w = sc.take<double>(k);
  double* d_d = sc.take<double>(k);
  int* d_perm = sc.take<int>(k);
  int* d_info = sc.take<int>(4);
  zval* gws = sc.take<zval>(gemm_ws_bytes(k, k, k) / sizeof(zval) + 1);
  bse::form_m_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(g2, mm, (int)k);
  check_launch(ctx);
  bse::hermitize_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(mm, (int)k);
  check_launch(ctx);
  CUDA_OK(cudaMemcpyAsync(tmp, mm, kk * sizeof(zval), cudaMemcpyDeviceToDevice, ctx->stream));
  heevd(ctx, tmp, (int)k, d_w, false, d_info);
  std::vector<double> hw(k);
  to_host(ctx, hw.data(), d_w, k);
  double lmm = INFINITY;
  for (double v : hw) lmm = std::min(lmm, std::fabs(v));
  if (h_lam_min_m) *h_lam_min_m = lmm;
  bse::diag_real_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(mm, (int)k, 1e-12, d_d);
  check_launch(ctx);
  capture_kk(ctx, 0, w, k);
  capture_kk(ctx, 2, mm, k);
  if (ctx->rr_capture)
    CUDA_OK(cudaMemcpyAsync(ctx->rr_capture + 4 * kk, d_d, k * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  bse::offdiag_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(mm, tmp, (int)k);
  check_launch(ctx);
  // g = (g0 - off W) / d
  zgemm<bse::OPA_N>(ctx, k, k, k, -1.0, tmp, k, w, k, 1.0, g, k, gws);
  bse::rowscale_inv_kernel<<<grid1d(kk), 256, 0, ctx->stream>>>(g, (int)k, d_d);
  check_launch(ctx);
  capture_kk(ctx, 3, g, k);
  // direct.py:102-116: general eigensolver, ascending real parts (stable)
  size_t dws = 0, hws = 0;
  SOLVER_OK(cusolverDnXgeev_bufferSize(ctx->solver, ctx->params, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR,
                                       k, CUDA_C_64F, g, k, CUDA_C_64F, d_ev, CUDA_C_64F, nullptr, 1, CUDA_C_64F, y, k,
                                       CUDA_C_64F, &dws, &hws));
  void* dbuf = solver_ws(ctx, dws);
  void* hbuf = host_ws(ctx, std::max<size_t>(hws, 16));
  SOLVER_OK(cusolverDnXgeev(ctx->solver, ctx->params, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, k,
                            CUDA_C_64F, g, k, CUDA_C_64F, d_ev, CUDA_C_64F, nullptr, 1, CUDA_C_64F, y, k, CUDA_C_64F,
                            dbuf, dws, hbuf, hws, d_info));
  int* info = reinterpret_cast<int*>(pinned(ctx, 1));
  CUDA_OK(cudaMemcpyAsync(info, d_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  if (*info != 0) throw BseError(BSE_ENUMERICAL, "general eigensolver failed (info " + std::to_string(*info) + ")");
  std::vector<double> ev(2 * k);
  to_host(ctx, ev.data(), reinterpret_cast<double*>(d_ev), 2 * k);
  std::vector<int> order(k);
  std::iota(order.begin(), order.end(), 0);
  for (int64_t i = 0; i < k; ++i)
    if (!std::isfinite(ev[2 * i]) || !std::isfinite(ev[2 * i + 1]))
      throw BseError(BSE_ENUMERICAL, "general eigensolver returned non-finite eigenvalues");
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ev[2 * a] < ev[2 * b]; });
  for (int64_t i = 0; i < k; ++i) h_lam[i] = ev[2 * order[i]];
  {
    std::vector<double> tmpd((k + 1) / 2 + 1);
    std::memcpy(tmpd.data(), order.data(), sizeof(int) * k);
    to_device(ctx, reinterpret_cast<double*>(d_perm), tmpd.data(), (k + 1) / 2);
  }
  bse::gather_cols_kernel<<<dim3(1, (unsigned)k), 256, 0, ctx->stream>>>(y, k, yperm, k, k, d_perm);
  check_launch(ctx);
}

int bse_rr_backup(bse_ctx* ctx, const void* d_ab, const void* d_sd, int64_t lda, int64_t m, const void* d_q,
                  int64_t ldq, int64_t k, double* h_lam, void* d_vout, int64_t ldvout, double* h_lam_min_m) {
  return guarded(ctx, [&] {
    if (k == 0) return;
    if (!d_ab && !rs_active(ctx, d_ab, m))
      throw BseError(BSE_EVALIDATION, "null operator: a planes-only operator needs bse_set_rs_planes(ctx, NULL, m, g, ldg)");
    const int64_t n = 2 * m;
    const zval* q = static_cast<const zval*>(d_q);
    zval* vout = static_cast<zval*>(d_vout);
    const size_t kk = (size_t)k * k;
    const size_t gwsb = std::max({gemm_ws_bytes(k, k, n), gemm_ws_bytes(k, k, m), gemm_ws_bytes(n, k, k)});
    const bool rs = (k > 1 || !d_ab) && rs_active(ctx, d_ab, m);
    Scratch sc(ctx, al(n * k * sizeof(zval)) + 4 * al(kk * sizeof(zval)) + al(k * 8) + gwsb + backup_ws_bytes(k) +
                        (rs ? al(n * k * sizeof(zval)) : 0));
    zval* t = sc.take<zval>(n * k);
    zval* fold = rs ? sc.take<zval>(n * k) : nullptr;
    zval* w = sc.take<zval>(kk);
    zval* g2 = sc.take<zval>(kk);
    zval* g = sc.take<zval>(kk);
    zval* yperm = sc.take<zval>(kk);
    double* d_nrm = sc.take<double>(k);
    zval* gws = sc.take<zval>(gwsb / sizeof(zval) + 1);
    // rayleigh_ritz.py:160-168
    apply_h(ctx, d_ab, lda, m, q, ldq, t, n, k, 1.0, d_sd, fold);
    zgemm<bse::OPA_C>(ctx, k, k, n, 1.0, q, ldq, t, n, 0.0, w, k, gws);
    zgemm<bse::OPA_C>(ctx, k, k, m, 1.0, q + m, ldq, q + m, ldq, 0.0, g2, k, gws);
    // g0 = Q^H (S T) = Q1^H T1 - Q2^H T2
    zgemm<bse::OPA_C>(ctx, k, k, m, 1.0, q, ldq, t, n, 0.0, g, k, gws);
    zgemm<bse::OPA_C>(ctx, k, k, m, -1.0, q + m, ldq, t + m, n, 1.0, g, k, gws);
    backup_pencil(ctx, g, w, g2, k, h_lam, yperm, h_lam_min_m, sc);
    zgemm<bse::OPA_N>(ctx, n, k, k, 1.0, q, ldq, yperm, k, 0.0, vout, ldvout, gws);
    bse::colnorm_kernel<<<(int)k, 256, 0, ctx->stream>>>(vout, ldvout, n, d_nrm);
    check_launch(ctx);
    bse::colscale_inv_kernel<<<dim3(grid1d(n, 256, 64), (unsigned)k), 256, 0, ctx->stream>>>(vout, ldvout, n, d_nrm);
    check_launch(ctx);
  });
}

int bse_rr_backup_pencil(bse_ctx* ctx, void* d_g0, const void* d_w, void* d_g2, int64_t k, double* h_lam,
                         void* d_y, double* h_lam_min_m) {
  return guarded(ctx, [&] {
    if (k <= 0) return;
    Scratch sc(ctx, backup_ws_bytes(k));
    backup_pencil(ctx, static_cast<zval*>(d_g0), static_cast<const zval*>(d_w), static_cast<zval*>(d_g2), k, h_lam,
                  static_cast<zval*>(d_y), h_lam_min_m, sc);
  });
}

int bse_lanczos_sweep(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, const void* h_start, int steps,
                      double* h_alpha, double* h_beta, int* h_count) {
  return guarded(ctx, [&] {
    const int64_t n = 2 * m;
    const int nb = grid1d(n, 256, 296);
    if (!d_ab && !rs_active(ctx, d_ab, m))
      throw BseError(BSE_EVALIDATION, "null operator: a planes-only operator needs bse_set_rs_planes(ctx, NULL, m, g, ldg)");
    Scratch sc(ctx, 7 * al(n * sizeof(zval)) + al((nb + 2) * 8) + al(64));
    zval* start = sc.take<zval>(n);
    zval* q = sc.take<zval>(n);
    zval* qold = sc.take<zval>(n);
    zval* z = sc.take<zval>(n);
    zval* w = sc.take<zval>(n);
    zval* gv = sc.take<zval>(n);
    zval* fold = d_ab ? nullptr : sc.take<zval>(n);  // planes-only operator: the matvec on the planes
    double* part = sc.take<double>(nb + 2);
    to_device(ctx, reinterpret_cast<double*>(start), static_cast<const double*>(h_start), 2 * n);
    auto sdot = [&](const zval* x, const zval* y) {
      bse::sdot_partial_kernel<<<nb, 256, 0, ctx->stream>>>(x, y, n, m, 1, part);
      check_launch(ctx);
      bse::sum_reduce_kernel<<<1, 256, 0, ctx->stream>>>(part, nb, part + nb);
      check_launch(ctx);
      double h = 0.0;
      to_host(ctx, &h, part + nb, 1);
      return h;
    };
    auto scale_div = [&](zval* out, const zval* in, double s) {
      // out = in / s  (division, as numpy's x / beta)
      CUDA_OK(cudaMemcpyAsync(out, in, n * sizeof(zval), cudaMemcpyDeviceToDevice, ctx->stream));
      to_device(ctx, part + nb + 1, &s, 1);
      bse::colscale_inv_kernel<<<dim3(grid1d(n, 256, 148), 1), 256, 0, ctx->stream>>>(out, n, n, part + nb + 1);
      check_launch(ctx);
    };
    // lanczos.py:58-66
    apply_h(ctx, d_ab, lda, m, start, n, gv, n, 1, 1.0, nullptr, fold);
    const double norm2 = sdot(gv, start);
    if (!(norm2 > 0))
      throw BseError(BSE_EINDEFINITE, "start vector has non-positive S*H norm; matrix is not definite");
    const double sc0 = std::sqrt(norm2);
    scale_div(q, start, sc0);
    scale_div(z, gv, sc0);
    CUDA_OK(cudaMemsetAsync(qold, 0, n * sizeof(zval), ctx->stream));
    double beta_prev = 0.0, amax = 0.0;
    int na = 0, nbeta = 0;
    for (int j = 0; j < steps; ++j) {
      const double alpha = sdot(z, z);  // lanczos.py:72
      h_alpha[na++] = alpha;
      amax = std::max(amax, std::fabs(alpha));
      if (j == steps - 1) break;
      bse::lincomb3_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(w, z, 1.0, q, -alpha, qold, -beta_prev, n);
      check_launch(ctx);
      apply_h(ctx, d_ab, lda, m, w, n, gv, n, 1, 1.0, nullptr, fold);
      const double beta2 = sdot(gv, w);
      const double running = std::max({1.0, amax, beta_prev});
      if (beta2 <= (1e-14 * running) * (1e-14 * running)) break;  // lanczos.py:79-81
      const double beta = std::sqrt(beta2);
      h_beta[nbeta++] = beta;
      std::swap(qold, q);
      scale_div(q, w, beta);
      scale_div(z, gv, beta);
      beta_prev = beta;
    }
    *h_count = na;
  });
}

int bse_is_definite(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, int* h_definite) {
  return guarded(ctx, [&] {
    const int64_t n = 2 * m;
    Scratch sc(ctx, al((size_t)n * n * sizeof(zval)) + al(64));
    zval* sh = sc.take<zval>((size_t)n * n);
    int* d_info = sc.take<int>(4);
    bse::materialize_sh_kernel<<<grid1d(n * n), 256, 0, ctx->stream>>>(static_cast<const zval*>(d_ab), lda, m, sh);
    check_launch(ctx);
    *h_definite = potrf(ctx, sh, (int)n, CUBLAS_FILL_MODE_LOWER, d_info) == 0 ? 1 : 0;
  });
}

bse::HopArgs tile_args(const bse_hop_tile_args* t) {
  bse::HopArgs a{};
  a.pa = static_cast<const zval*>(t->pa);
  a.pb = static_cast<const zval*>(t->pb);
  a.sa = static_cast<const zval*>(t->sa);
  a.sb = static_cast<const zval*>(t->sb);
  a.lda = t->lda;
  a.mr = (int)t->mr;
  a.kc = (int)t->kc;
  a.x1 = static_cast<const zval*>(t->x1);
  a.x2 = static_cast<const zval*>(t->x2);
  a.ldx = t->ldx;
  a.k = (int)t->k;
  a.y1 = static_cast<zval*>(t->y1);
  a.y2 = static_cast<zval*>(t->y2);
  a.ldy = t->ldy;
  a.s1 = static_cast<const zval*>(t->s1);
  a.s2 = static_cast<const zval*>(t->s2);
  a.lds = t->lds;
  a.shift_lo = (int)t->shift_lo;
  a.shift_hi = (int)t->shift_hi;
  a.shift = t->shift;
  a.shift_col = t->d_shift_col;
  a.p1 = static_cast<const zval*>(t->p1);
  a.p2 = static_cast<const zval*>(t->p2);
  a.ldp = t->ldp;
  a.alpha = t->alpha;
  a.beta = t->beta;
  a.low_sign = t->low_sign;
  return a;
}

int bse_hop_tile(bse_ctx* ctx, const bse_hop_tile_args* t) {
  return guarded(ctx, [&] {
    if (!t) throw BseError(BSE_EVALIDATION, "null args");
    if (t->k <= 0 || t->mr <= 0) return;
    bse::HopArgs a = tile_args(t);
    if (a.beta != 0.0 && (!a.p1 || !a.p2)) throw BseError(BSE_EVALIDATION, "beta != 0 needs p1/p2");
    if ((a.shift != 0.0 || a.shift_col) && a.shift_hi > a.shift_lo && (!a.s1 || !a.s2))
      throw BseError(BSE_EVALIDATION, "shift needs s1/s2");
    if (a.kc <= 0) throw BseError(BSE_EVALIDATION, "empty contraction");
    const bool plain = a.beta == 0.0 && !a.shift_col && (a.shift == 0.0 || a.shift_hi <= a.shift_lo);
    if (a.k == 1 && plain)
      launch_gemv(ctx, a);
    else if (t->filter)
      launch_filter_hop(ctx, a);
    else
      launch_hop<HopMain, bse::HOP_AXPBY>(ctx, a);
  });
}

int bse_hop_tile_rs(bse_ctx* ctx, const bse_hop_tile_args* t, const void* d_g, int64_t ldg) {
  return guarded(ctx, [&] {
    if (!t || !d_g) throw BseError(BSE_EVALIDATION, "null args");
    if (t->k <= 0 || t->mr <= 0) return;
    bse::HopArgs a = tile_args(t);
    if (a.kc <= 0) throw BseError(BSE_EVALIDATION, "empty contraction");
    if (ldg < a.mr || (ldg & 1)) throw BseError(BSE_EVALIDATION, "ldg must be even and >= mr");
    if (a.low_sign != 1.0) throw BseError(BSE_EVALIDATION, "the real-split product has no S-flip (low_sign 1)");
    if (a.beta != 0.0 && (!a.p1 || !a.p2)) throw BseError(BSE_EVALIDATION, "beta != 0 needs p1/p2");
    if ((a.shift != 0.0 || a.shift_col) && a.shift_hi > a.shift_lo && (!a.s1 || !a.s2))
      throw BseError(BSE_EVALIDATION, "shift needs s1/s2");
    if (ctx->ham_flags & BSE_HAM_B_ZERO) throw BseError(BSE_EVALIDATION, "the real-split product needs B != 0");
    rs_product(ctx, a, static_cast<const double*>(d_g), ldg);
  });
}

int bse_set_push_targets(bse_ctx* ctx, void* const* y_bases, int n) {
  return guarded(ctx, [&] {
    if (n < 0 || n > 4 || (n > 0 && !y_bases)) throw BseError(BSE_EVALIDATION, "push targets: 0..4 base pointers");
    for (int r = 0; r < n; ++r)
      if (!y_bases[r]) throw BseError(BSE_EVALIDATION, "null push target");
    ctx->push_n = n;
    for (int r = 0; r < 4; ++r) ctx->push_base[r] = r < n ? static_cast<zval*>(y_bases[r]) : nullptr;
  });
}

int bse_group_sum(bse_ctx* ctx, const void* d_inbox, int64_t slot_stride, int nslot, void* d_y, int64_t count) {
  return guarded(ctx, [&] {
    if (count <= 0) return;
    if (!d_inbox || !d_y || nslot < 1 || slot_stride < count) throw BseError(BSE_EVALIDATION, "group sum arguments");
    const int blocks = (int)std::min<int64_t>((count + 255) / 256, 148 * 16);
    bse::group_sum_kernel<<<blocks, 256, 0, ctx->stream>>>(static_cast<const zval*>(d_inbox), slot_stride, nslot,
                                                          static_cast<zval*>(d_y), count);
    check_launch(ctx);
  });
}

int bse_hop_tile_rs_t(bse_ctx* ctx, const bse_hop_tile_args* t, const void* d_g, int64_t ldg) {
  return guarded(ctx, [&] {
    if (!t || !d_g) throw BseError(BSE_EVALIDATION, "null args");
    if (t->k <= 0 || t->mr <= 0) return;
    bse::HopArgs a = tile_args(t);
    if (a.kc <= 0) throw BseError(BSE_EVALIDATION, "empty contraction");
    if (ldg < a.kc || (ldg & 1)) throw BseError(BSE_EVALIDATION, "ldg must be even and >= kc (the plane rows)");
    if (a.low_sign != 1.0) throw BseError(BSE_EVALIDATION, "the real-split product has no S-flip (low_sign 1)");
    if (a.beta != 0.0 && (!a.p1 || !a.p2)) throw BseError(BSE_EVALIDATION, "beta != 0 needs p1/p2");
    if ((a.shift != 0.0 || a.shift_col) && a.shift_hi > a.shift_lo && (!a.s1 || !a.s2))
      throw BseError(BSE_EVALIDATION, "shift needs s1/s2");
    if (ctx->ham_flags & BSE_HAM_B_ZERO) throw BseError(BSE_EVALIDATION, "the real-split product needs B != 0");
    rs_product<true>(ctx, a, static_cast<const double*>(d_g), ldg);
  });
}

int bse_rs_fold(bse_ctx* ctx, const void* d_src, void* d_dst, int64_t ld, int64_t rows, int64_t k, double scale,
                double scale2) {
  return guarded(ctx, [&] {
    if (rows < 0 || k < 0 || ld < 2 * rows) throw BseError(BSE_EVALIDATION, "bad shapes");
    if (rows == 0 || k == 0) return;
    bse::rs_fold_kernel<<<grid1d(rows * k, 256, 148 * 16), 256, 0, ctx->stream>>>(
        static_cast<const zval*>(d_src), static_cast<zval*>(d_dst), ld, ld, rows, k, scale, scale2);
    check_launch(ctx);
  });
}

int bse_chol_rinv(bse_ctx* ctx, void* d_g, int64_t k, double shift, void* d_rinv, double* d_rdiag, int* h_info) {
  return guarded(ctx, [&] {
    if (k <= 0) return;
    Scratch sc(ctx, al(64));
    int* d_info = sc.take<int>(4);
    zval* g = static_cast<zval*>(d_g);
    bse::hermitize_kernel<<<grid1d(k * k), 256, 0, ctx->stream>>>(g, (int)k);
    check_launch(ctx);
    if (shift != 0.0) {
      bse::add_diag_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(g, (int)k, shift);
      check_launch(ctx);
    }
    const int info = potrf(ctx, g, (int)k, CUBLAS_FILL_MODE_UPPER, d_info);
    *h_info = info;
    if (info != 0) return;
    if (d_rdiag) {
      bse::absdiag_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(g, (int)k, d_rdiag);
      check_launch(ctx);
    }
    zval* rinv = static_cast<zval*>(d_rinv);
    bse::set_identity_kernel<<<grid1d(k * k), 256, 0, ctx->stream>>>(rinv, (int)k);
    check_launch(ctx);
    const cuDoubleComplex z1 = make_cuDoubleComplex(1.0, 0.0);
    BLAS_OK(cublasZtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)k,
                        (int)k, &z1, cz(g), (int)k, cz(rinv), (int)k));
  });
}

int bse_rr_pencil(bse_ctx* ctx, void* d_w, void* d_g2, int64_t k, double* h_lam, void* d_wvec, double* h_lam_min_m) {
  return guarded(ctx, [&] {
    if (k <= 0) return;
    Scratch sc(ctx, pencil_ws_bytes(k) + 4096);
    rr_pencil(ctx, static_cast<zval*>(d_w), static_cast<zval*>(d_g2), k, h_lam, static_cast<zval*>(d_wvec),
              h_lam_min_m, sc);
  });
}

int bse_rr_pencil_part(bse_ctx* ctx, int part, void* d_w, void* d_g2, int64_t k, double* h_lam, void* d_wvec,
                       double* h_lam_min_m) {
  return guarded(ctx, [&] {
    if (part != 1 && part != 2) throw BseError(BSE_EVALIDATION, "part must be 1 or 2");
    if (k <= 0) return;
    Scratch sc(ctx, pencil_ws_bytes(k) + 4096);
    rr_pencil(ctx, static_cast<zval*>(d_w), static_cast<zval*>(d_g2), k, h_lam, static_cast<zval*>(d_wvec),
              h_lam_min_m, sc, part);
  });
}

int bse_resid_partial(bse_ctx* ctx, const void* d_u, int64_t ldu, const void* d_v, int64_t ldv, int64_t rows,
                      int64_t half, int64_t k, const double* d_uscale, const double* d_lam, double* d_out) {
  return guarded(ctx, [&] {
    if (k <= 0) return;
    bse::resid_from_rr_kernel<<<(int)k, 256, 0, ctx->stream>>>(static_cast<const zval*>(d_u), ldu,
                                                               static_cast<const zval*>(d_v), ldv, rows, half,
                                                               d_uscale, d_lam, d_out);
    check_launch(ctx);
  });
}

int bse_colnorm2(bse_ctx* ctx, const void* d_x, int64_t rows, int64_t k, int64_t ldx, double* d_out) {
  return guarded(ctx, [&] {
    if (k <= 0) return;
    bse::frob2_kernel<<<(int)k, 256, 0, ctx->stream>>>(static_cast<const zval*>(d_x), ldx, rows, d_out);
    check_launch(ctx);
  });
}

int bse_colscale_rsqrt(bse_ctx* ctx, void* d_x, int64_t rows, int64_t k, int64_t ldx, const double* d_norm2) {
  return guarded(ctx, [&] {
    if (k <= 0 || rows <= 0) return;
    Scratch sc(ctx, al(k * 8));
    double* nrm = sc.take<double>(k);
    bse::sqrt_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(d_norm2, nrm, (int)k);
    check_launch(ctx);
    bse::colscale_inv_kernel<<<dim3(grid1d(rows, 256, 64), (unsigned)k), 256, 0, ctx->stream>>>(
        static_cast<zval*>(d_x), ldx, rows, nrm);
    check_launch(ctx);
  });
}

int bse_defect(bse_ctx* ctx, const void* d_g, int64_t k, double* h_out) {
  return guarded(ctx, [&] {
    if (k <= 0) {
      *h_out = 0.0;
      return;
    }
    Scratch sc(ctx, al(1024 * 8));
    double* part = sc.take<double>(1024);
    *h_out = defect_to_host(ctx, static_cast<const zval*>(d_g), (int)k, part);
  });
}

int bse_sflip(bse_ctx* ctx, const void* d_x, int64_t ldx, void* d_y, int64_t ldy, int64_t half, int64_t k) {
  return guarded(ctx, [&] {
    if (k <= 0 || half <= 0) return;
    bse::sflip_copy_kernel<<<grid1d(2 * half * k), 256, 0, ctx->stream>>>(static_cast<const zval*>(d_x), ldx,
                                                                           static_cast<zval*>(d_y), ldy, half, k);
    check_launch(ctx);
  });
}

int bse_c64_prepare(bse_ctx* ctx, const void* d_ab, int64_t lda, int64_t m, void* d_pplanes) {
  return guarded(ctx, [&] {
    if (m <= 0) return;
    const int64_t mp = pad4(m), plane = m * 2 * mp;
    float* pl = static_cast<float*>(d_pplanes);
    const zval* ab = static_cast<const zval*>(d_ab);
    bse::c64::p_planes_kernel<<<grid1d(plane, 256, 148 * 32), 256, 0, ctx->stream>>>(
        ab, ab + m * lda, lda, (int)m, (int)m, (int)mp, pl, pl + plane, pl + 2 * plane, pl + 3 * plane);
    check_launch(ctx);
  });
}

int bse_c64_tile_planes(bse_ctx* ctx, const void* d_src_a, const void* d_src_b, int64_t lds, int64_t mo, int64_t kc,
                        void* d_pplanes) {
  return guarded(ctx, [&] {
    if (mo <= 0 || kc <= 0) return;
    if (lds < kc) throw BseError(BSE_EVALIDATION, "bad shapes");
    const int64_t mp = pad4(kc), plane = mo * 2 * mp;
    float* pl = static_cast<float*>(d_pplanes);
    bse::c64::p_planes_kernel<<<grid1d(plane, 256, 148 * 32), 256, 0, ctx->stream>>>(
        static_cast<const zval*>(d_src_a), static_cast<const zval*>(d_src_b), lds, (int)mo, (int)kc, (int)mp, pl,
        pl + plane, pl + 2 * plane, pl + 3 * plane);
    check_launch(ctx);
  });
}

int bse_c64_tile_step(bse_ctx* ctx, const bse_c64_tile_args* t) {
  return guarded(ctx, [&] {
    if (!t) throw BseError(BSE_EVALIDATION, "null args");
    if (t->k <= 0 || t->mo <= 0) return;
    if (t->kc <= 0) throw BseError(BSE_EVALIDATION, "bad shapes");
    C64Step st{};
    st.mo = t->mo;
    st.kc = t->kc;
    st.k = t->k;
    float* xs[8];
    plane_set(static_cast<float*>(const_cast<void*>(t->x)), t->kc, t->k, xs);
    for (int q = 0; q < 8; ++q) st.x[q] = xs[q];
    float* ps[8];
    if (t->prev && t->beta != 0.0) {
      plane_set(static_cast<float*>(const_cast<void*>(t->prev)), t->mo, t->k, ps);
      for (int q = 0; q < 4; ++q) st.prev[q] = ps[q];
    }
    float* os[8];
    plane_set(static_cast<float*>(t->out), t->mo, t->k, os);
    for (int q = 0; q < 8; ++q) st.out[q] = os[q];
    st.alpha = t->alpha;
    st.beta = t->beta;
    st.shift = t->shift;
    st.shift_lo = t->shift_lo;
    st.shift_hi = t->shift_hi;
    st.s_off = t->s_off;
    st.raw = t->raw != 0;
    bse::c64::Maps maps;
    c64_p_maps(maps, static_cast<const float*>(t->pplanes), t->mo, t->kc);
    c64_step(ctx, maps, st);
  });
}

int bse_c64_split(bse_ctx* ctx, const void* d_raw, int64_t rows, int64_t k, void* d_planes) {
  return guarded(ctx, [&] {
    if (rows <= 0 || k <= 0) return;
    const int64_t blk = 2 * pad4(rows) * k;
    const float* raw = static_cast<const float*>(d_raw);
    float* os[8];
    plane_set(static_cast<float*>(d_planes), rows, k, os);
    bse::c64::Planes8 q;
    for (int i = 0; i < 8; ++i) q.p[i] = os[i];
    bse::c64::split_planes_kernel<<<grid1d(blk, 256, 148 * 32), 256, 0, ctx->stream>>>(raw, raw + blk, (int)rows,
                                                                                       (int)pad4(rows), (int)k, q);
    check_launch(ctx);
  });
}

int bse_c64_to_planes(bse_ctx* ctx, const void* d_v, int64_t ldv, int64_t rows, int64_t k, void* d_planes) {
  return guarded(ctx, [&] {
    if (rows <= 0 || k <= 0) return;
    float* os[8];
    plane_set(static_cast<float*>(d_planes), rows, k, os);
    bse::c64::Planes8 q;
    for (int i = 0; i < 8; ++i) q.p[i] = os[i];
    bse::c64::to_planes_kernel<<<grid1d(2 * pad4(rows) * k, 256, 148 * 32), 256, 0, ctx->stream>>>(
        static_cast<const zval*>(d_v), ldv, (int)rows, (int)pad4(rows), (int)k, q);
    check_launch(ctx);
  });
}

int bse_c64_from_planes(bse_ctx* ctx, const void* d_planes, int64_t rows, int64_t k, void* d_v, int64_t ldv) {
  return guarded(ctx, [&] {
    if (rows <= 0 || k <= 0) return;
    float* os[8];
    plane_set(static_cast<float*>(const_cast<void*>(d_planes)), rows, k, os);
    bse::c64::from_planes_kernel<<<grid1d(2 * rows * k, 256, 148 * 32), 256, 0, ctx->stream>>>(
        os[0], os[1], os[2], os[3], (int)rows, (int)pad4(rows), (int)k, static_cast<zval*>(d_v), ldv);
    check_launch(ctx);
  });
}

int bse_chebyshev_filter_c64(bse_ctx* ctx, const void* d_pplanes, int64_t m, void* d_v, int64_t ldv, int64_t k, int deg,
                             double c, double e, double s, void* d_work) {
  return guarded(ctx, [&] {
    if (deg < 2 || deg % 2) throw BseError(BSE_EVALIDATION, "filter degree must be even and >= 2");
    if (!(e > 0)) throw BseError(BSE_EVALIDATION, "filter half width must be positive");
    if (k <= 0 || m <= 0) return;
    const int64_t mp = pad4(m), blk = 2 * mp * k;
    float* w = static_cast<float*>(d_work);
    float* bufs[3][8];
    for (int b = 0; b < 3; ++b)
      for (int q = 0; q < 8; ++q) bufs[b][q] = w + (int64_t)(8 * b + q) * blk;
    bse::c64::Planes8 p0;
    for (int q = 0; q < 8; ++q) p0.p[q] = bufs[0][q];
    bse::c64::to_planes_kernel<<<grid1d(blk, 256, 148 * 32), 256, 0, ctx->stream>>>(
        static_cast<const zval*>(d_v), ldv, (int)m, (int)mp, (int)k, p0);
    check_launch(ctx);
    bse::c64::Maps maps;
    c64_p_maps(maps, static_cast<const float*>(d_pplanes), m, m);
    auto step_on = [&](int in, int pv, int out, double alpha, double beta) {
      C64Step st{};
      st.mo = st.kc = m;
      st.k = k;
      for (int q = 0; q < 8; ++q) st.x[q] = bufs[in][q];
      for (int q = 0; q < 4; ++q) st.prev[q] = pv >= 0 ? bufs[pv][q] : nullptr;
      for (int q = 0; q < 8; ++q) st.out[q] = bufs[out][q];
      st.alpha = alpha;
      st.beta = beta;
      st.shift = c;
      st.shift_lo = 0;
      st.shift_hi = m;
      st.s_off = 0;
      c64_step(ctx, maps, st);
    };
    // chebyshev.py:58-74 on three rotating plane blocks
    const double sigma1 = e / (s - c);
    double sigma = sigma1;
    int prev = 0, cur = 1;
    step_on(0, -1, 1, sigma1 / e, 0.0);
    for (int step = 2; step <= deg; ++step) {
      const double sigma_new = 1.0 / (2.0 / sigma1 - sigma);
      const int nxt = 3 - prev - cur;
      step_on(cur, prev, nxt, 2.0 * sigma_new / e, sigma * sigma_new);
      prev = cur;
      cur = nxt;
      sigma = sigma_new;
    }
    const int64_t n = 2 * m;
    bse::c64::from_planes_kernel<<<grid1d(n * k, 256, 148 * 32), 256, 0, ctx->stream>>>(
        bufs[cur][0], bufs[cur][1], bufs[cur][2], bufs[cur][3], (int)m, (int)mp, (int)k, static_cast<zval*>(d_v), ldv);
    check_launch(ctx);
  });
}

int bse_complex_normals(bse_ctx* ctx, void* d_out, uint64_t seed, int64_t start_index, int64_t count) {
  return guarded(ctx, [&] {
    if (count <= 0) return;
    bse::complex_normals_kernel<<<grid1d(count, 256, 148 * 32), 256, 0, ctx->stream>>>(static_cast<zval*>(d_out), seed,
                                                                                       start_index, count);
    check_launch(ctx);
  });
}

int bse_complex_normals_t(bse_ctx* ctx, void* d_out, uint64_t seed, int64_t rows, int64_t cols) {
  return guarded(ctx, [&] {
    if (rows <= 0 || cols <= 0) return;
    bse::complex_normals_t_kernel<<<grid1d(rows * cols, 256, 148 * 32), 256, 0, ctx->stream>>>(
        static_cast<zval*>(d_out), seed, rows, cols);
    check_launch(ctx);
  });
}

int bse_symmetrize(bse_ctx* ctx, void* d_a, int64_t m, int64_t lda, int conj) {
  return guarded(ctx, [&] {
    if (m <= 0) return;
    bse::symmetrize_kernel<<<grid1d(m * m, 256, 148 * 32), 256, 0, ctx->stream>>>(static_cast<zval*>(d_a), lda, m, conj);
    check_launch(ctx);
  });
}

int bse_scale_shift(bse_ctx* ctx, void* d_a, int64_t m, int64_t lda, double scale, double shift, int conj) {
  return guarded(ctx, [&] {
    if (m <= 0) return;
    bse::scale_shift_kernel<<<grid1d(m * m, 256, 148 * 32), 256, 0, ctx->stream>>>(static_cast<zval*>(d_a), lda, m,
                                                                                  scale, shift, conj);
    check_launch(ctx);
  });
}

int bse_eigvalsh(bse_ctx* ctx, const void* d_a, int64_t k, int64_t lda, double* h_w) {
  return guarded(ctx, [&] {
    if (k <= 0) return;
    Scratch sc(ctx, al((size_t)k * k * sizeof(zval)) + al(k * 8) + al(64));
    zval* a = sc.take<zval>((size_t)k * k);
    double* d_w = sc.take<double>(k);
    int* d_info = sc.take<int>(4);
    CUDA_OK(cudaMemcpy2DAsync(a, sizeof(zval) * k, d_a, sizeof(zval) * lda, sizeof(zval) * k, (size_t)k,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    heevd(ctx, a, (int)k, d_w, false, d_info);
    to_host(ctx, h_w, d_w, k);
  });
}

}  // extern "C"
