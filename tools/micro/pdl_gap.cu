// Per-boundary cost of a chain of dependent small kernels in a CUDA graph, with and without
// programmatic dependent launch (PDL): nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_gap.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(const float* __restrict__ in, float* __restrict__ out, int n, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] * 1.0001f + 1.f;
}

int main() {
    const int n = 1 << 16, chain = 40, reps = 200;
    float *a, *b;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4);
    cudaMemset(a, 0, n * 4);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < chain; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl ? 1 : 0;
            cudaLaunchKernelEx(&cfg, step_kernel, (const float*)(i & 1 ? b : a), (i & 1 ? a : b), n, pdl);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, st);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("pdl=%d  %d-kernel chain: %.2f us per graph, %.3f us per kernel  (%s)\n", pdl, chain, 1000.f * ms / reps,
               1000.f * ms / reps / chain, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
