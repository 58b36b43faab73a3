// Microbenchmark: MUFU tanh throughput (f32 vs f16x2 vs bf16x2) on sm_100a.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
__global__ void k_f32(float* out, int iters) {
  float x = threadIdx.x * 1e-3f, a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a0)); asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a1));
      asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a2)); asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
__global__ void k_f16x2(float* out, int iters) {
  unsigned a0 = 0x3c003c00u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(a0)); asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(a1));
      asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(a2)); asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(a3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(a0 ^ a1 ^ a2 ^ a3);
}
__global__ void k_bf16x2(float* out, int iters) {
  unsigned a0 = 0x3f803f80u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(a0)); asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(a1));
      asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(a2)); asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(a3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(a0 ^ a1 ^ a2 ^ a3);
}
__global__ void k_ex2(float* out, int iters) {
  float x = threadIdx.x * 1e-3f, a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
__global__ void k_hfma2(float* out, int iters) {
  __half2 a0 = __floats2half2_rn(0.1f*threadIdx.x, 1.f), a1 = a0, a2 = a0, a3 = a0, m = __floats2half2_rn(0.999f, 0.999f), c = __floats2half2_rn(0.001f, 0.001f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { a0 = __hfma2(a0, m, c); a1 = __hfma2(a1, m, c); a2 = __hfma2(a2, m, c); a3 = __hfma2(a3, m, c); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = __low2float(a0) + __low2float(a1) + __low2float(a2) + __low2float(a3);
}
__global__ void k_ffma(float* out, int iters) {
  float a0 = 0.1f*threadIdx.x, a1 = a0+1, a2 = a0+2, a3 = a0+3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { a0 = fmaf(a0, 0.999f, 0.001f); a1 = fmaf(a1, 0.999f, 0.001f); a2 = fmaf(a2, 0.999f, 0.001f); a3 = fmaf(a3, 0.999f, 0.001f); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
template <class K> void run(const char* name, K k, float* d, int ops_per_thread_iter) {
  int blocks = 148 * 8, threads = 256, iters = 4096;
  k<<<blocks, threads>>>(d, 16); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(blocks) * threads * iters * 32;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_clk_sm = ops / (ms * 1e-3) / 148 / (clk * 1e3);
  printf("%-10s %8.3f ms  %.2f Tinstr/s  %.1f instr/clk/SM (@%d MHz nominal) x%d values\n", name, ms, ops / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000, ops_per_thread_iter);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  run("tanh.f32", k_f32, d, 1); run("tanh.f16x2", k_f16x2, d, 2); run("tanh.bf16x2", k_bf16x2, d, 2);
  run("ex2.f32", k_ex2, d, 1); run("hfma2", k_hfma2, d, 2); run("ffma", k_ffma, d, 1);
  return 0;
}
