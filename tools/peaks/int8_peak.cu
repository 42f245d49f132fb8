// INT8 tensor-core roofline denominator for the Ozaki-scheme GEMM (ozgemm.cu) on B200:
// cuBLAS int8 x int8 -> int32 GEMM (IMMA / tcgen05 kind::i8 inside cuBLAS) at large square and
// at the power-product shape, best of repeated timings (CUDA events). One JSON object on stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int8_peak int8_peak.cu -lcublas
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
#define CB(x) do { cublasStatus_t s = (x); if (s != CUBLAS_STATUS_SUCCESS) { fprintf(stderr, "%s:%d cublas %d\n", __FILE__, __LINE__, (int)s); exit(1);} } while (0)

static double tops(cublasHandle_t h, int m, int n, int k, void* A, void* B, void* C) {
  const int alpha = 1, beta = 0;
  auto run = [&] {
    CB(cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, m, n, k, &alpha, A, CUDA_R_8I, k, B, CUDA_R_8I, k, &beta, C,
                    CUDA_R_32I, m, CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT));
  };
  for (int i = 0; i < 3; ++i) run();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) run();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    if (ms / 5 < best) best = ms / 5;
  }
  return 2.0 * m * n * (double)k / (best * 1e-3) / 1e12;
}

int main() {
  const size_t big = (size_t)16384 * 16384;
  void *A, *B, *C;
  CK(cudaMalloc(&A, big)); CK(cudaMalloc(&B, big)); CK(cudaMalloc(&C, big * 4));
  CK(cudaMemset(A, 1, big)); CK(cudaMemset(B, 1, big));
  cublasHandle_t h; CB(cublasCreate(&h));
  const double sq = tops(h, 8192, 8192, 8192, A, B, C);
  const double zr = tops(h, 131072 / 16, 512, 1024, A, B, C);  // 8192 x 512 x 1024 slice of the Z shape
  printf("{\"cublas_int8_8192_tops\": %.1f, \"cublas_int8_8192x512x1024_tops\": %.1f, \"nominal_int8_dense_tops\": 4500}\n", sq, zr);
  return 0;
}
