// FP64 roofline denominators for the FGFRFT hot path on B200 (sm_100a).
// Measures: DFMA issue peak, DMMA (mma.sync f64, m8n8k4 and m16n8k16) peak,
// cuBLAS DGEMM/ZGEMM throughput, and a streaming read / copy HBM figure.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu -lcublas
// Output: one JSON object on stdout.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cuComplex.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 123.456) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double2 acc = make_double2(0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p + i));
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 123.456) out[0] = acc.y;
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 64));
  const int iters = 4096;
  // DFMA: blocks x threads x iters x 16 fma x 2 flops
  int blocks = sms * 8, threads = 256;
  float t = time_ms([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); }, 5);
  double dfma_tf = (double)blocks * threads * iters * 16 * 2 / (t * 1e-3) / 1e12;
  // DMMA m8n8k4: per warp-instr 8*8*4 FMA
  t = time_ms([&] { dmma884_kernel<<<blocks, threads>>>(out, iters); }, 5);
  double dmma884_tf = (double)blocks * (threads / 32) * iters * 8 * (8 * 8 * 4) * 2 / (t * 1e-3) / 1e12;
  t = time_ms([&] { dmma16816_kernel<<<blocks, threads>>>(out, iters / 4); }, 5);
  double dmma16816_tf = (double)blocks * (threads / 32) * (iters / 4) * 4 * (16 * 8 * 16) * 2 / (t * 1e-3) / 1e12;

  // cuBLAS DGEMM / ZGEMM
  cublasHandle_t h; cublasCreate(&h);
  const int n = 8192;
  double *A, *B, *C;
  CK(cudaMalloc(&A, (size_t)n * n * 16)); CK(cudaMalloc(&B, (size_t)n * n * 16)); CK(cudaMalloc(&C, (size_t)n * n * 16));
  CK(cudaMemset(A, 0, (size_t)n * n * 16)); CK(cudaMemset(B, 0, (size_t)n * n * 16));
  double one = 1, zero = 0;
  t = time_ms([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n); }, 3);
  double dgemm_tf = 2.0 * n * n * (double)n / (t * 1e-3) / 1e12;
  cuDoubleComplex zone = make_cuDoubleComplex(1, 0), zzero = make_cuDoubleComplex(0, 0);
  const int nz = 4096;
  t = time_ms([&] { cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, nz, nz, nz, &zone, (cuDoubleComplex*)A, nz, (cuDoubleComplex*)B, nz, &zzero, (cuDoubleComplex*)C, nz); }, 3);
  double zgemm_tf = 8.0 * nz * nz * (double)nz / (t * 1e-3) / 1e12;
  // ZGEMM at the apply shape of config 2/3: N x B, K = N
  t = time_ms([&] { cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, 4096, 1024, 4096, &zone, (cuDoubleComplex*)A, 4096, (cuDoubleComplex*)B, 4096, &zzero, (cuDoubleComplex*)C, 4096); }, 3);
  double zgemm_apply_tf = 8.0 * 4096 * 1024 * 4096.0 / (t * 1e-3) / 1e12;

  // HBM: stream-read 4 GiB and copy 2 GiB
  size_t bytes = (size_t)4 << 30;
  double2* big; CK(cudaMalloc(&big, bytes)); CK(cudaMemset(big, 0, bytes));
  t = time_ms([&] { read_kernel<<<sms * 8, 512>>>(big, bytes / 16, out); }, 5);
  double read_gbs = bytes / (t * 1e-3) / 1e9;
  t = time_ms([&] { cudaMemcpyAsync((char*)big + bytes / 2, big, bytes / 2, cudaMemcpyDeviceToDevice); }, 5);
  double copy_gbs = bytes / (t * 1e-3) / 1e9;  // read + write bytes

  printf("{\"sms\": %d, \"dfma_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, "
         "\"cublas_dgemm_8192_tflops\": %.2f, \"cublas_zgemm_4096_tflops\": %.2f, \"cublas_zgemm_4096x1024x4096_tflops\": %.2f, "
         "\"hbm_read_gbs\": %.1f, \"hbm_copy_gbs\": %.1f}\n",
         sms, dfma_tf, dmma884_tf, dmma16816_tf, dgemm_tf, zgemm_tf, zgemm_apply_tf, read_gbs, copy_gbs);
  return 0;
}
