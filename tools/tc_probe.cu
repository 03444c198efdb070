// Probe: tcgen05 TF32 GEMM  C (M x N, fp32) = A (M x K, K-major) * B (N x K, K-major)^T
// TMA SW128 loads -> mbarrier pipeline -> tcgen05.mma (one elected thread) -> TMEM -> tcgen05.ld.
// Validates the descriptor encodings before they are used in the c64 filter kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2601_10557_b200/csrc/tc_common.cuh"

using namespace bse::tc;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s @%d: %s\n", cudaGetErrorString(e), __LINE__, #x);         \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int BM = 128, BN = 128, BKB = 32, STAGES = 4;
constexpr int TILE_A = BM * BKB * 4, TILE_B = BN * BKB * 4;

__global__ void __launch_bounds__(128, 1) tc_gemm(const __grid_constant__ CUtensorMap ma,
                                                  const __grid_constant__ CUtensorMap mb, float* C, int M, int N,
                                                  int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-align the tile region
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = base;
  unsigned char* sb = base + STAGES * TILE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * TILE_B);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BKB - 1) / BKB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
    prefetch_tmap(&ma);
    prefetch_tmap(&mb);
  }
  if (warp == 0) tmem_alloc(tslot, BN);  // BN fp32 columns x 128 lanes
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], TILE_A + TILE_B);
      tma_load_2d(sa + s * TILE_A, &ma, &full[s], kb * BKB, m0);
      tma_load_2d(sb + s * TILE_B, &mb, &full[s], kb * BKB, n0);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    constexpr uint32_t idesc = idesc_tf32(BM, BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      fence_after_sync();
      const uint32_t a0 = smem_addr(sa + s * TILE_A), b0 = smem_addr(sb + s * TILE_B);
#pragma unroll
      for (int kk = 0; kk < BKB / 8; ++kk)  // 8 tf32 = 32 bytes per UMMA K step
        mma_tf32(tmem, sdesc_k_sw128(a0 + kk * 32), sdesc_k_sw128(b0 + kk * 32), idesc, (kb | kk) != 0);
      mma_commit(&empty[s]);
    }
    mma_commit(done);
  }
  // epilogue: 4 warps x 32 TMEM lanes = 128 rows
  mbar_wait(done, 0);
  fence_after_sync();
  const int row = m0 + warp * 32 + lane;
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    if (row < M)
      for (int j = 0; j < 16; ++j)
        if (n0 + c + j < N) C[(size_t)row * N + n0 + c + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, BN);
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
  const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 256, K = argc > 3 ? atoi(argv[3]) : 512;
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
  CUtensorMap ma = make_map(da, M, K, BM), mb = make_map(db, N, K, BN);
  const size_t smem = 1024 + STAGES * (TILE_A + TILE_B) + 256;
  CK(cudaFuncSetAttribute(tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  tc_gemm<<<grid, 128, smem>>>(ma, mb, dc, M, N, K);
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
  printf("tc_gemm M=%d N=%d K=%d: max |err| %.3e (max |ref| %.3e, rel %.3e) -> %s\n", M, N, K, maxerr, maxref,
         maxerr / maxref, maxerr / maxref < 5e-3 ? "OK" : "FAIL");
  // throughput at a large shape
  const int LM = 8192, LN = 8192, LK = 8192;
  float *la, *lb, *lc;
  CK(cudaMalloc(&la, (size_t)LM * LK * 4));
  CK(cudaMalloc(&lb, (size_t)LN * LK * 4));
  CK(cudaMalloc(&lc, (size_t)LM * LN * 4));
  CK(cudaMemset(la, 0, (size_t)LM * LK * 4));
  CK(cudaMemset(lb, 0, (size_t)LN * LK * 4));
  CUtensorMap lma = make_map(la, LM, LK, BM), lmb = make_map(lb, LN, LK, BN);
  dim3 lgrid(LN / BN, LM / BM);
  tc_gemm<<<lgrid, 128, smem>>>(lma, lmb, lc, LM, LN, LK);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) tc_gemm<<<lgrid, 128, smem>>>(lma, lmb, lc, LM, LN, LK);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("tc_gemm 8192^3 tf32: %.3f ms, %.1f TFLOP/s\n", ms / 5, 2.0 * LM * LN * (double)LK * 5 / ms / 1e9);
  return 0;
}
