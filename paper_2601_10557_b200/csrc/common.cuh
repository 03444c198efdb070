// Shared device helpers for the sm_100a FP64 kernels.
//
// FP64 on B200: tcgen05.mma has no f64 kind, so the tensor path for double
// precision is the warp-level DMMA.8x8x4 (PTX mma.sync.m8n8k4.f64), measured
// at 37.1 TFLOP/s per GPU (profiles/fp64_peak.json).  Operands are staged
// global -> shared with cp.async (LDGSTS) multi-stage pipelines; complex
// values stay interleaved (re, im) so one LDS.128 yields both planes of a
// fragment element.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bse {

struct __align__(16) zval {
  double re, im;
};

// D = A(8x4, row) * B(4x8, col) + D ; lane (g = lane/4, t = lane%4) holds
// a = A[g][t], b = B[t][g], d = {D[g][2t], D[g][2t+1]}.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy; src_bytes = 0 zero-fills the destination (ragged edges).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}
// 8-byte async copy (X-side 3M sum planes)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// plain shared load of one complex (compiles to LDS.128)
__device__ __forceinline__ zval lds128(const zval* p) { return *p; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace bse
