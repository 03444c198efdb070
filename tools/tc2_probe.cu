// Probe: 2-SM tcgen05 TF32 GEMM (cta_group::2), C (M x N, fp32) = A (M x K) * B (N x K)^T, both
// K-major.  A CTA pair (cluster 2 x 1, M tiles along x) computes a 256 x N tile: each CTA stages its own
// 128 A rows and half of the N B rows; the leader CTA issues M = 256 UMMAs reading both CTAs'
// shared memory; each CTA's TMEM holds its 128 rows x N accumulator.  Validates the protocol
// (peer-masked TMA barrier, multicast commits, 2-SM TMEM allocation) and measures whether halving
// each SM's B-operand shared-memory reads lifts the N = 128 tf32 rate (c64.cuh is smem-read bound).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2601_10557_b200/csrc/tc_common.cuh"

using namespace bse::tc;

#define CK(x)                                                           \
  do {                                                                  \
    cudaError_t e = (x);                                                \
    if (e != cudaSuccess) {                                             \
      printf("CUDA %s @%d: %s\n", cudaGetErrorString(e), __LINE__, #x); \
      exit(1);                                                          \
    }                                                                   \
  } while (0)

constexpr int BM = 128, BN = 128, BKB = 32, STAGES = 4;  // BN = N of the pair's MMA; each CTA holds BN/2 B rows
constexpr int TILE_A = BM * BKB * 4, TILE_B = (BN / 2) * BKB * 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  const uint32_t b = smem_addr(bar) & 0xFEFFFFFFu;  // the leader CTA's barrier
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(b), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc ? 1u : 0u));
}
__device__ __forceinline__ void commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_addr(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__global__ void __launch_bounds__(192, 1)
    tc2_gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, float* C, int M, int N,
             int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = base;
  unsigned char* sb = base + STAGES * TILE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * TILE_B);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int m0 = blockIdx.x * BM;                           // this CTA's rows (pairs along x)
  const int n0 = blockIdx.y * BN + (int)rank * (BN / 2);    // this CTA's half of the B rows
  const int nk = (K + BKB - 1) / BKB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(tslot)), "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  fence_before_sync();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  fence_after_sync();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {  // TMA producer, both CTAs
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
      if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (TILE_A + TILE_B));  // both CTAs' bytes
      tma_load_2d_2sm(sa + s * TILE_A, &ma, &full[s], kb * BKB, m0);
      tma_load_2d_2sm(sb + s * TILE_B, &mb, &full[s], kb * BKB, n0);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {  // MMA issuer: leader only
    const uint32_t idesc = idesc_tf32(2 * BM, BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      fence_after_sync();
      const uint32_t a0 = smem_addr(sa + s * TILE_A), b0 = smem_addr(sb + s * TILE_B);
#pragma unroll
      for (int kk = 0; kk < BKB / 8; ++kk)
        mma_tf32_2sm(tmem, sdesc_k_sw128(a0 + kk * 32), sdesc_k_sw128(b0 + kk * 32), idesc, (kb | kk) != 0);
      commit_2sm(&empty[s]);
    }
    commit_2sm(done);
  }
  if (warp >= 2) {  // epilogue: 4 warps x 32 TMEM lanes = this CTA's 128 rows, all BN columns
    mbar_wait(done, 0);
    fence_after_sync();
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
      if (row < M)
        for (int j = 0; j < 16; ++j)
          if (blockIdx.y * BN + c + j < N) C[(size_t)row * N + blockIdx.y * BN + c + j] = v[j];
    }
  }
  fence_before_sync();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(const float* g, int rows, int K, int box_rows) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {BKB, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)g, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("cuTensorMapEncodeTiled failed %d\n", (int)r);
    exit(1);
  }
  return map;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 512, N = argc > 2 ? atoi(argv[2]) : 256, K = argc > 3 ? atoi(argv[3]) : 512;
  std::vector<float> a((size_t)M * K), b((size_t)N * K), c((size_t)M * N);
  srand(1);
  for (auto& x : a) x = (rand() / (float)RAND_MAX) - 0.5f;
  for (auto& x : b) x = (rand() / (float)RAND_MAX) - 0.5f;
  float *da, *db, *dc;
  CK(cudaMalloc(&da, a.size() * 4));
  CK(cudaMalloc(&db, b.size() * 4));
  CK(cudaMalloc(&dc, c.size() * 4));
  CK(cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dc, 0, c.size() * 4));
  CUtensorMap ma = make_map(da, M, K, BM), mb = make_map(db, N, K, BN / 2);
  const size_t smem = 1024 + STAGES * (TILE_A + TILE_B) + 256;
  CK(cudaFuncSetAttribute(tc2_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(((M + BM - 1) / BM + 1) / 2 * 2, (N + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = grid;
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = -1;
  cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclusters, tc2_gemm, &cfg);
  printf("max active clusters: %d (%s)\n", nclusters, cudaGetErrorString(oe));
  CK(cudaLaunchKernelEx(&cfg, tc2_gemm, ma, mb, dc, M, N, K));
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(c.data(), dc, c.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)a[(size_t)i * K + k] * b[(size_t)j * K + k];
      maxerr = fmax(maxerr, fabs(s - c[(size_t)i * N + j]));
      maxref = fmax(maxref, fabs(s));
    }
  printf("tc2_gemm M=%d N=%d K=%d: max |err| %.3e (max |ref| %.3e, rel %.3e) -> %s\n", M, N, K, maxerr, maxref,
         maxerr / maxref, maxerr / maxref < 5e-3 ? "OK" : "FAIL");
  const int LM = 8192, LN = 8192, LK = 8192;
  float *la, *lb, *lc;
  CK(cudaMalloc(&la, (size_t)LM * LK * 4));
  CK(cudaMalloc(&lb, (size_t)LN * LK * 4));
  CK(cudaMalloc(&lc, (size_t)LM * LN * 4));
  CK(cudaMemset(la, 0, (size_t)LM * LK * 4));
  CK(cudaMemset(lb, 0, (size_t)LN * LK * 4));
  CUtensorMap lma = make_map(la, LM, LK, BM), lmb = make_map(lb, LN, LK, BN / 2);
  dim3 lgrid(LM / BM, LN / BN);
  cfg.gridDim = lgrid;
  CK(cudaLaunchKernelEx(&cfg, tc2_gemm, lma, lmb, lc, LM, LN, LK));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) CK(cudaLaunchKernelEx(&cfg, tc2_gemm, lma, lmb, lc, LM, LN, LK));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("tc2_gemm 8192^3 tf32 (2-SM, N=%d): %.3f ms, %.1f TFLOP/s\n", BN, ms / 5, 2.0 * LM * LN * (double)LK * 5 / ms / 1e9);
  return 0;
}
