// Legacy warp-level mma.sync throughput on sm_100a (TF32 m16n8k8 and FP32 FFMA for reference).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tf32_kernel(float* out, int iters) {
    float d[8][4] = {};
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_kernel(float* out, int iters) {
    float x[16];
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 0.001f + j;
    const float a = 1.0001f, b = 0.9999f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
    }
    float s = 0;
    for (int j = 0; j < 16; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 4, threads = 256, iters = 4096;
    tf32_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    tf32_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * (blocks * threads / 32);
    printf("mma.sync tf32 m16n8k8: %.1f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
    ffma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * iters * (double)(blocks * threads);
    printf("ffma fp32: %.1f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
    return 0;
}
