// Row LayerNorm forward / backward (Tape::layer_norm, proj/src/tape.cpp:84-100
// and its VJP :581-617; eps 1e-5): the normalisation after the merge projection
// and in the transformer blocks.
//
// One warp per row (persistent grid-stride over rows); a lane holds C/32
// elements as 8-byte bf16 vectors (C in {128, 256, 384, 512, 768, 1024}).
// Mean, then the centred variance, as the reference (two passes over
// registers), fp32 statistics saved for the backward.  dgamma / dbeta: per-warp fp32 partials in registers, written per
// warp and summed in a fixed order by a second kernel (deterministic).
#include "common.cuh"

namespace affmae_b200 {

constexpr float kLnEpsF = 1e-5f;
constexpr int kLnWarps = 8;

__device__ __forceinline__ void ln_bf8(const uint2& v, float (&f)[4]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
__device__ __forceinline__ uint2 ln_pack(const float (&f)[4]) {
    uint2 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 2; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}

// VPL: 4-element (8-byte) bf16 vectors per lane (C = 128 * VPL)
template <int VPL>
__global__ void __launch_bounds__(kLnWarps * 32) ln_fwd_kernel(const uint2* __restrict__ x, const float* __restrict__ gamma,
                                                               const float* __restrict__ beta, int64_t rows,
                                                               uint2* __restrict__ y, float2* __restrict__ stats) {
    constexpr int C = 128 * VPL;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = int64_t(blockIdx.x) * kLnWarps + (threadIdx.x >> 5), ws = int64_t(gridDim.x) * kLnWarps;
    for (int64_t r = w0; r < rows; r += ws) {
        float v[VPL][4];
#pragma unroll
        for (int j = 0; j < VPL; ++j) ln_bf8(__ldg(x + r * (C / 4) + j * 32 + lane), v[j]);
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) s += v[j][i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float mu = s / float(C);
        float q = 0.f;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) q = fmaf(v[j][i] - mu, v[j][i] - mu, q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        const float inv = rsqrtf(q / float(C) + kLnEpsF);
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            const int c0 = (j * 32 + lane) * 4;
            float o8[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) o8[i] = fmaf(__ldg(gamma + c0 + i), (v[j][i] - mu) * inv, __ldg(beta + c0 + i));
            y[r * (C / 4) + j * 32 + lane] = ln_pack(o8);
        }
        if (lane == 0) stats[r] = make_float2(mu, inv);
    }
}

template <int VPL>
__global__ void __launch_bounds__(kLnWarps * 32) ln_bwd_kernel(const uint2* __restrict__ x, const float* __restrict__ gamma,
                                                               const float2* __restrict__ stats,
                                                               const uint2* __restrict__ dy, int64_t rows,
                                                               uint2* __restrict__ dx, float* __restrict__ part) {
    constexpr int C = 128 * VPL;
    const int lane = threadIdx.x & 31;
    const int64_t wid = int64_t(blockIdx.x) * kLnWarps + (threadIdx.x >> 5), ws = int64_t(gridDim.x) * kLnWarps;
    float dg[VPL][4], db[VPL][4];
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) dg[j][i] = db[j][i] = 0.f;
    for (int64_t r = wid; r < rows; r += ws) {
        const float2 st = __ldg(stats + r);
        float xh[VPL][4], g[VPL][4];
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            float xv[4];
            ln_bf8(__ldg(x + r * (C / 4) + j * 32 + lane), xv);
            ln_bf8(__ldg(dy + r * (C / 4) + j * 32 + lane), g[j]);
            const int c0 = (j * 32 + lane) * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                xh[j][i] = (xv[i] - st.x) * st.y;
                const float dxh = g[j][i] * __ldg(gamma + c0 + i);
                s1 += dxh;
                s2 = fmaf(dxh, xh[j][i], s2);
                dg[j][i] = fmaf(g[j][i], xh[j][i], dg[j][i]);
                db[j][i] += g[j][i];
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        const float m1 = s1 / float(C), m2 = s2 / float(C);
        if (dx) {
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                const int c0 = (j * 32 + lane) * 4;
                float o8[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) o8[i] = st.y * (g[j][i] * __ldg(gamma + c0 + i) - m1 - xh[j][i] * m2);
                dx[r * (C / 4) + j * 32 + lane] = ln_pack(o8);
            }
        }
    }
    // per-warp partials [warp][2][C]
    float* pw = part + wid * 2 * C;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
        const int c0 = (j * 32 + lane) * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            pw[c0 + i] = dg[j][i];
            pw[C + c0 + i] = db[j][i];
        }
    }
}

__global__ void ln_param_grad_kernel(const float* __restrict__ part, int64_t nwarps, int C,
                                     float* __restrict__ dgamma, float* __restrict__ dbeta) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 2 * C) return;
    float s = 0.f;
    for (int64_t w = 0; w < nwarps; ++w) s += part[w * 2 * C + c];
    if (c < C) {
        if (dgamma) dgamma[c] += s;
    } else if (dbeta) {
        dbeta[c - C] += s;
    }
}

static unsigned ln_blocks(int64_t rows) {
    return unsigned(std::max<int64_t>(1, std::min<int64_t>((rows + kLnWarps - 1) / kLnWarps, 4 * kNumSMs)));
}

size_t layernorm_bwd_workspace(int64_t rows, int64_t cols) {
    return size_t(ln_blocks(rows)) * kLnWarps * 2 * size_t(cols) * 4 + 256;
}

int layernorm_fwd(const void* x, const float* gamma, const float* beta, int64_t rows, int64_t cols, void* y,
                  float* stats, void* stream) {
    if (!x || !gamma || !beta || !y || !stats) return fail(AFFMAE_ECONFIG, "layer_norm: null pointer");
    if (rows < 0 || cols < 1) return fail(AFFMAE_ECONFIG, "layer_norm: bad shape");
    if (rows == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const auto* xv = static_cast<const uint2*>(x);
    auto* yv = static_cast<uint2*>(y);
    auto* s2 = reinterpret_cast<float2*>(stats);
    const unsigned nb = ln_blocks(rows);
    switch (cols) {
        case 128: ln_fwd_kernel<1><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, beta, rows, yv, s2); break;
        case 256: ln_fwd_kernel<2><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, beta, rows, yv, s2); break;
        case 384: ln_fwd_kernel<3><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, beta, rows, yv, s2); break;
        case 512: ln_fwd_kernel<4><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, beta, rows, yv, s2); break;
        case 768: ln_fwd_kernel<6><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, beta, rows, yv, s2); break;
        case 1024: ln_fwd_kernel<8><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, beta, rows, yv, s2); break;
        default: return fail(AFFMAE_EUNSUPPORTED, "layer_norm: cols must be 128, 256, 384, 512, 768 or 1024");
    }
    AFFMAE_LAUNCH_CHECK("ln_fwd_kernel");
    return AFFMAE_OK;
}

int layernorm_bwd(const void* x, const float* gamma, const float* stats, const void* dy, int64_t rows, int64_t cols,
                  void* dx, float* dgamma, float* dbeta, void* workspace, size_t ws_bytes, void* stream) {
    if (!x || !gamma || !stats || !dy) return fail(AFFMAE_ECONFIG, "layer_norm bwd: null pointer");
    if (rows < 0 || cols < 1) return fail(AFFMAE_ECONFIG, "layer_norm bwd: bad shape");
    if (!workspace || ws_bytes < layernorm_bwd_workspace(rows, cols))
        return fail(AFFMAE_ECONFIG, "layer_norm bwd: workspace too small");
    if (rows == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const auto* xv = static_cast<const uint2*>(x);
    const auto* gv = static_cast<const uint2*>(dy);
    auto* dxv = static_cast<uint2*>(dx);
    const auto* s2 = reinterpret_cast<const float2*>(stats);
    float* part = static_cast<float*>(workspace);
    const unsigned nb = ln_blocks(rows);
    switch (cols) {
        case 128: ln_bwd_kernel<1><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, s2, gv, rows, dxv, part); break;
        case 256: ln_bwd_kernel<2><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, s2, gv, rows, dxv, part); break;
        case 384: ln_bwd_kernel<3><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, s2, gv, rows, dxv, part); break;
        case 512: ln_bwd_kernel<4><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, s2, gv, rows, dxv, part); break;
        case 768: ln_bwd_kernel<6><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, s2, gv, rows, dxv, part); break;
        case 1024: ln_bwd_kernel<8><<<nb, kLnWarps * 32, 0, st>>>(xv, gamma, s2, gv, rows, dxv, part); break;
        default: return fail(AFFMAE_EUNSUPPORTED, "layer_norm: cols must be 128, 256, 384, 512, 768 or 1024");
    }
    ln_param_grad_kernel<<<unsigned((2 * cols + 255) / 256), 256, 0, st>>>(part, int64_t(nb) * kLnWarps, int(cols),
                                                                        dgamma, dbeta);
    AFFMAE_LAUNCH_CHECK("ln_bwd_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
