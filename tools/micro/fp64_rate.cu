// FP64 vs FP32 add/mul throughput on this GPU (8 independent chains per thread).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chains(T* out, int iters, T a, T b) {
    T x[8];
    for (int i = 0; i < 8; ++i) x[i] = T(threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = x[i] * a + b;
    T s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename T>
float run(int iters) {
    T* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(T));
    chains<T><<<148 * 8, 256>>>(out, 10, T(0.999), T(0.001));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chains<T><<<148 * 8, 256>>>(out, iters, T(0.999), T(0.001));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    return ms;
}
int main() {
    const int iters = 4096;
    const double fma = double(148) * 8 * 256 * iters * 8;
    float m32 = run<float>(iters), m64 = run<double>(iters);
    printf("fp32 FMA: %.3f ms  %.1f TFLOP/s\n", m32, 2 * fma / m32 / 1e9);
    printf("fp64 FMA: %.3f ms  %.1f TFLOP/s\n", m64, 2 * fma / m64 / 1e9);
    return 0;
}
