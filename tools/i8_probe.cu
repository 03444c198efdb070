// Probe: tcgen05 INT8 GEMM  C (M x N, s32) = A (M x K, s8, K-major) * B (N x K, s8, K-major)^T
// TMA SW128 loads -> mbarrier ring -> tcgen05.mma.kind::i8 (one elected thread) -> TMEM -> tcgen05.ld.
// Validates the S8/S32 instruction descriptor and measures the int8 tensor rate on B200 before the
// integer-slice (Ozaki) filter is built on it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

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

constexpr int BM = 128, BN = 256, BKB = 128, STAGES = 4;  // BKB in bytes = int8 elements
constexpr int TILE_A = BM * BKB, TILE_B = BN * BKB;

__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  return (2u << 4)                      // c_format = S32
         | (1u << 7)                    // a_format = signed 8 bit
         | (1u << 10)                   // b_format = signed 8 bit
         | ((uint32_t)(N >> 3) << 17)   // N >> 3
         | ((uint32_t)(M >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc ? 1u : 0u));
}

__global__ void __launch_bounds__(128, 1) i8_gemm(const __grid_constant__ CUtensorMap ma,
                                                  const __grid_constant__ CUtensorMap mb, int* C, int M, int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
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
  }
  if (warp == 0) tmem_alloc(tslot, BN);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], TILE_A + TILE_B);
      tma_load_2d(sa + s * TILE_A, &ma, &full[s], kb * BKB, m0);
      tma_load_2d(sb + s * TILE_B, &mb, &full[s], kb * BKB, n0);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_s8(BM, BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      fence_after_sync();
      const uint32_t a0 = smem_addr(sa + s * TILE_A), b0 = smem_addr(sb + s * TILE_B);
#pragma unroll
      for (int kk = 0; kk < BKB / 32; ++kk)
        mma_i8(tmem, sdesc_k_sw128(a0 + kk * 32), sdesc_k_sw128(b0 + kk * 32), idesc, (kb | kk) != 0);
      mma_commit(&empty[s]);
    }
    mma_commit(done);
  }
  mbar_wait(done, 0);
  fence_after_sync();
  const int row = m0 + warp * 32 + lane;
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    if (row < M)
      for (int j = 0; j < 16; ++j)
        if (n0 + c + j < N) C[(size_t)row * N + n0 + c + j] = __float_as_int(v[j]);
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

static CUtensorMap make_map(const void* g, int rows, int K, int box_rows) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {BKB, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)g, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("cuTensorMapEncodeTiled failed %d\n", (int)r);
    exit(1);
  }
  return map;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 512, K = argc > 3 ? atoi(argv[3]) : 1024;
  std::vector<signed char> a((size_t)M * K), b((size_t)N * K);
  std::vector<int> c((size_t)M * N);
  srand(1);
  for (auto& x : a) x = (signed char)((rand() % 255) - 127);
  for (auto& x : b) x = (signed char)((rand() % 255) - 127);
  void *da, *db;
  int* dc;
  CK(cudaMalloc(&da, a.size()));
  CK(cudaMalloc(&db, b.size()));
  CK(cudaMalloc(&dc, c.size() * 4));
  CK(cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dc, 0, c.size() * 4));
  CUtensorMap ma = make_map(da, M, K, BM), mb = make_map(db, N, K, BN);
  const size_t smem = 1024 + STAGES * (TILE_A + TILE_B) + 256;
  CK(cudaFuncSetAttribute(i8_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  i8_gemm<<<grid, 128, smem>>>(ma, mb, dc, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(c.data(), dc, c.size() * 4, cudaMemcpyDeviceToHost));
  long long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long long s = 0;
      for (int k = 0; k < K; ++k) s += (long long)a[(size_t)i * K + k] * b[(size_t)j * K + k];
      if (s != c[(size_t)i * N + j]) ++bad;
    }
  printf("i8_gemm M=%d N=%d K=%d: %lld mismatches -> %s\n", M, N, K, bad, bad ? "FAIL" : "OK (exact)");
  const int LM = 16384, LN = 16384, LK = 16384;
  void *la, *lb;
  int* lc;
  CK(cudaMalloc(&la, (size_t)LM * LK));
  CK(cudaMalloc(&lb, (size_t)LN * LK));
  CK(cudaMalloc(&lc, (size_t)LM * LN * 4));
  CK(cudaMemset(la, 1, (size_t)LM * LK));
  CK(cudaMemset(lb, 1, (size_t)LN * LK));
  CUtensorMap lma = make_map(la, LM, LK, BM), lmb = make_map(lb, LN, LK, BN);
  dim3 lgrid(LN / BN, LM / BM);
  i8_gemm<<<lgrid, 128, smem>>>(lma, lmb, lc, LM, LN, LK);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) i8_gemm<<<lgrid, 128, smem>>>(lma, lmb, lc, LM, LN, LK);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("i8_gemm %d^3 s8: %.3f ms, %.1f TOP/s\n", LM, ms / 5, 2.0 * LM * LN * (double)LK * 5 / ms / 1e9);
  return 0;
}
