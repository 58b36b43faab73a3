// Decoder-side row ops:
//   * NormClampOp (proj/src/pipeline.cpp:75-127): y = x * min(1, limit / |x|) per
//     row, VJP dx = g (|x| <= limit) or (limit/|x|)(g - (g.x / |x|^2) x);
//   * the reconstruction loss (Tape::mse, proj/src/tape.cpp:431-446, VJP :694-707;
//     Model::loss_parts, pipeline.cpp:581-600): mean squared error of the
//     prediction rows against the target patches of the masked cells, gathered
//     by index on the device (no host-side target tensor).
// Warp per row, fp32 accumulation; the loss sum is a two-level fixed-order
// reduction (deterministic).
#include "common.cuh"

namespace affmae_b200 {

constexpr int kDecWarps = 8;

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kDecWarps * 32) norm_clamp_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                                        int64_t rows, int d, float limit,
                                                                        __nv_bfloat16* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t ws = int64_t(gridDim.x) * kDecWarps;
    for (int64_t r = int64_t(blockIdx.x) * kDecWarps + (threadIdx.x >> 5); r < rows; r += ws) {
        const __nv_bfloat16* xr = x + r * d;
        float s = 0.f;
        for (int j = lane; j < d; j += 32) {
            const float v = __bfloat162float(xr[j]);
            s = fmaf(v, v, s);
        }
        const float nrm = sqrtf(warp_sum_f(s));
        const float f = nrm > limit ? limit / nrm : 1.f;
        for (int j = lane; j < d; j += 32) y[r * d + j] = __float2bfloat16(__bfloat162float(xr[j]) * f);
    }
}

__global__ void __launch_bounds__(kDecWarps * 32) norm_clamp_bwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                                        const __nv_bfloat16* __restrict__ g,
                                                                        int64_t rows, int d, float limit,
                                                                        __nv_bfloat16* __restrict__ dx) {
    const int lane = threadIdx.x & 31;
    const int64_t ws = int64_t(gridDim.x) * kDecWarps;
    for (int64_t r = int64_t(blockIdx.x) * kDecWarps + (threadIdx.x >> 5); r < rows; r += ws) {
        const __nv_bfloat16* xr = x + r * d;
        const __nv_bfloat16* gr = g + r * d;
        float s = 0.f, dot = 0.f;
        for (int j = lane; j < d; j += 32) {
            const float v = __bfloat162float(xr[j]), gv = __bfloat162float(gr[j]);
            s = fmaf(v, v, s);
            dot = fmaf(gv, v, dot);
        }
        s = warp_sum_f(s);
        dot = warp_sum_f(dot);
        const float nrm = sqrtf(s);
        // ACCUMULATES into dx (NormClampOp::backward, pipeline.cpp:104-125: dx += J^T g)
        if (nrm <= limit) {
            for (int j = lane; j < d; j += 32)
                dx[r * d + j] = __float2bfloat16(__bfloat162float(dx[r * d + j]) + __bfloat162float(gr[j]));
        } else {
            const float f = limit / nrm, c = dot / s;
            for (int j = lane; j < d; j += 32)
                dx[r * d + j] = __float2bfloat16(__bfloat162float(dx[r * d + j]) +
                                                 f * (__bfloat162float(gr[j]) - c * __bfloat162float(xr[j])));
        }
    }
}

// loss partial per block: sum over its rows of (pred - target[cell])^2
__global__ void __launch_bounds__(kDecWarps * 32) masked_mse_kernel(const __nv_bfloat16* __restrict__ pred,
                                                                    const float* __restrict__ patches,
                                                                    const int32_t* __restrict__ cells, int64_t rows,
                                                                    int p, float scale, __nv_bfloat16* __restrict__ dpred,
                                                                    float* __restrict__ part) {
    __shared__ float red[kDecWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ws = int64_t(gridDim.x) * kDecWarps;
    float acc = 0.f;
    for (int64_t r = int64_t(blockIdx.x) * kDecWarps + warp; r < rows; r += ws) {
        const float* t = patches + int64_t(__ldg(cells + r)) * p;
        for (int j = lane; j < p; j += 32) {
            const float dlt = __bfloat162float(pred[r * p + j]) - __ldg(t + j);
            acc = fmaf(dlt, dlt, acc);
            if (dpred) dpred[r * p + j] = __float2bfloat16(scale * dlt);  // d(mean)/d pred = 2 dlt / numel
        }
    }
    acc = warp_sum_f(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int w = 0; w < kDecWarps; ++w) s += red[w];
        part[blockIdx.x] = s;
    }
}
__global__ void mse_final_kernel(const float* __restrict__ part, int n, float inv_numel, float* __restrict__ loss) {
    __shared__ float red[32];
    float s = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    s = warp_sum_f(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        *loss = t * inv_numel;
    }
}

static unsigned dec_blocks(int64_t rows) {
    return unsigned(std::max<int64_t>(1, std::min<int64_t>((rows + kDecWarps - 1) / kDecWarps, 4 * kNumSMs)));
}

int norm_clamp_fwd(const void* x, int64_t rows, int64_t d, double limit, void* y, void* stream) {
    if (!x || !y) return fail(AFFMAE_ECONFIG, "norm_clamp: null pointer");
    if (rows < 0 || d < 1 || d > INT32_MAX) return fail(AFFMAE_ECONFIG, "norm_clamp: bad shape");
    if (rows == 0) return AFFMAE_OK;
    norm_clamp_fwd_kernel<<<dec_blocks(rows), kDecWarps * 32, 0, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), rows, int(d), float(limit), static_cast<__nv_bfloat16*>(y));
    AFFMAE_LAUNCH_CHECK("norm_clamp_fwd_kernel");
    return AFFMAE_OK;
}

int norm_clamp_bwd(const void* x, const void* g, int64_t rows, int64_t d, double limit, void* dx, void* stream) {
    if (!x || !g || !dx) return fail(AFFMAE_ECONFIG, "norm_clamp bwd: null pointer");
    if (rows < 0 || d < 1 || d > INT32_MAX) return fail(AFFMAE_ECONFIG, "norm_clamp bwd: bad shape");
    if (rows == 0) return AFFMAE_OK;
    norm_clamp_bwd_kernel<<<dec_blocks(rows), kDecWarps * 32, 0, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g), rows, int(d), float(limit),
        static_cast<__nv_bfloat16*>(dx));
    AFFMAE_LAUNCH_CHECK("norm_clamp_bwd_kernel");
    return AFFMAE_OK;
}

size_t masked_mse_workspace(int64_t rows) { return size_t(dec_blocks(rows)) * 4 + 256; }

int masked_mse(const void* pred, const float* patches, const int32_t* cells, int64_t rows, int64_t p, float* loss,
               void* dpred, float dloss, void* workspace, size_t ws_bytes, void* stream) {
    if (!pred || !patches || !cells || !loss) return fail(AFFMAE_ECONFIG, "masked_mse: null pointer");
    if (rows < 1 || p < 1 || p > INT32_MAX) return fail(AFFMAE_ECONFIG, "masked_mse: bad shape");
    if (!workspace || ws_bytes < masked_mse_workspace(rows)) return fail(AFFMAE_ECONFIG, "masked_mse: workspace");
    cudaStream_t st = as_stream(stream);
    const unsigned nb = dec_blocks(rows);
    const double numel = double(rows) * double(p);
    masked_mse_kernel<<<nb, kDecWarps * 32, 0, st>>>(static_cast<const __nv_bfloat16*>(pred), patches, cells, rows,
                                                     int(p), float(2.0 * dloss / numel),
                                                     static_cast<__nv_bfloat16*>(dpred), static_cast<float*>(workspace));
    mse_final_kernel<<<1, 1024, 0, st>>>(static_cast<float*>(workspace), int(nb), float(1.0 / numel), loss);
    AFFMAE_LAUNCH_CHECK("masked_mse");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
