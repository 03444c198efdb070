// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA
// register-only throughput, plus cuBLAS DGEMM/ZGEMM at large shapes.
// Used once to fix the roofline denominator (MEASURED_PEAKS.json has no FP64 figure).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cuComplex.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
  double acc[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = 0.0; acc[c][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(a, acc[c], b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    dmma_loop<8><<<grid, block>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * 8 * iters * (double)grid.x * warps;
    printf("DMMA m8n8k4 warps/blk=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", warps, grid.x, flops / ms / 1e9, ms);
  }
  for (int warps : {8, 16, 32}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<8><<<grid, block>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)grid.x * warps * 32;
    printf("DFMA warps/blk=%d: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  // sustained DMMA for ~4 s
  {
    dim3 grid(sms * 2), block(32 * 8);
    int iters = 20000;
    cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    for (; reps < 400; ++reps) dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * 8 * iters * (double)grid.x * 8 * reps;
    printf("DMMA sustained (%d launches, %.1f s): %.2f TFLOP/s\n", reps, ms / 1e3, flops / ms / 1e9);
  }
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {4096, 8192, 16384}) {
    double *A, *B, *C; size_t bytes = (size_t)n * n * 8;
    CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes);
    double one = 1, zero = 0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    CK(cudaDeviceSynchronize());
    int reps = n >= 16384 ? 3 : 10;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cuBLAS DGEMM n=%d: %.2f TFLOP/s\n", n, 2.0 * n * n * (double)n * reps / ms / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // ZGEMM at the filter shape: M=m, K=2m, N=2k (m=20000, k=1200) and C2 (m=10000,k=600)
  for (int cfg = 0; cfg < 2; ++cfg) {
    int m = cfg ? 20000 : 10000, k = cfg ? 1200 : 600;
    int M = m, K = 2 * m, N = 2 * k;
    cuDoubleComplex *A, *B, *C;
    CK(cudaMalloc(&A, (size_t)M * K * 16)); CK(cudaMalloc(&B, (size_t)K * N * 16)); CK(cudaMalloc(&C, (size_t)M * N * 16));
    cudaMemset(A, 0, (size_t)M * K * 16); cudaMemset(B, 0, (size_t)K * N * 16);
    cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &one, A, M, B, K, &zero, C, M);
    CK(cudaDeviceSynchronize());
    int reps = 5;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &one, A, M, B, K, &zero, C, M);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cuBLAS ZGEMM M=%d N=%d K=%d: %.2f TFLOP/s (8MNK model), %.2f ms/call\n", M, N, K, 8.0 * M * (double)N * K * reps / ms / 1e9, ms / reps);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  return 0;
}
