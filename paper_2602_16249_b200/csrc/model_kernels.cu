// Row / elementwise kernels of the device-resident training step (model.cu): the pieces of
// Model::encode / decode / deep_sup (proj/src/pipeline.cpp:373-579) that are not GEMMs,
// attention, interpolation or merge ops.
//
//   * LayerNorm over an fp32 (residual stream) or bf16 row with an optional fused residual
//     add, and its VJP fused with the residual-gradient accumulation
//     (Tape::layer_norm, proj/src/tape.cpp:84-100 / VJP :581-617; eps 1e-5);
//   * the positional MLP's first layer (pos_encode, pipeline.cpp:373-377: 2 -> 16, GELU);
//   * the merge scorer's output unit (pipeline.cpp:453-454: 16 -> 1, sigmoid);
//   * the decoder's offset head + NormClampOp (pipeline.cpp:75-127, :505-509);
//   * mask-cell compaction, patch / coordinate gathers, casts, residual adds, column sums.
//
// Parameter-gradient reductions are deterministic: per-block partials in a fixed layout,
// then a fixed-order sum (colsum_partials_kernel) that ACCUMULATES into the gradient arena.
#include "common.cuh"
#include "model_kernels.h"

namespace affmae_b200 {
namespace mk {

constexpr float kLnEps = 1e-5f;
constexpr int kRowWarps = 8;

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
    const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
    const float pdf = 0.39894228040143268f * expf(-0.5f * x * x);
    return cdf + x * pdf;
}

__device__ __forceinline__ float2 ld2(const float* p, int64_t i) { return *reinterpret_cast<const float2*>(p + i); }
__device__ __forceinline__ float2 ld2(const __nv_bfloat16* p, int64_t i) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p + i));
}
__device__ __forceinline__ void st2(float* p, int64_t i, float2 v) { *reinterpret_cast<float2*>(p + i) = v; }
__device__ __forceinline__ void st2(__nv_bfloat16* p, int64_t i, float2 v) {
    *reinterpret_cast<__nv_bfloat162*>(p + i) = __floats2bfloat162_rn(v.x, v.y);
}

static unsigned row_blocks(int64_t rows, int per_block, int cap = 4 * kNumSMs) {
    return unsigned(std::max<int64_t>(1, std::min<int64_t>((rows + per_block - 1) / per_block, cap)));
}

// ------------------------------------------------------------------ LayerNorm
// One warp per row; lane l holds columns 2(l + 32 j), j < V  (C = 64 V).
template <int V, typename XT>
__global__ void __launch_bounds__(kRowWarps * 32)
    ln_fwd_kernel(const XT* __restrict__ x, const __nv_bfloat16* __restrict__ add, float* __restrict__ xo,
                  __nv_bfloat16* __restrict__ xo_bf, const float* __restrict__ gamma, const float* __restrict__ beta,
                  int64_t rows, __nv_bfloat16* __restrict__ y, float2* __restrict__ stats) {
    constexpr int C = 64 * V;
    const int lane = threadIdx.x & 31;
    for (int64_t r = int64_t(blockIdx.x) * kRowWarps + (threadIdx.x >> 5); r < rows;
         r += int64_t(gridDim.x) * kRowWarps) {
        float2 v[V];
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int64_t i = r * C + 2 * (lane + 32 * j);
            v[j] = ld2(x, i);
            if (add) {
                const float2 a = ld2(add, i);
                v[j].x += a.x;
                v[j].y += a.y;
            }
            if (xo) st2(xo, i, v[j]);
            if (xo_bf) st2(xo_bf, i, v[j]);
            s += v[j].x + v[j].y;
        }
        s = warp_sum(s);
        const float mu = s / float(C);
        float q = 0.f;
#pragma unroll
        for (int j = 0; j < V; ++j) q += (v[j].x - mu) * (v[j].x - mu) + (v[j].y - mu) * (v[j].y - mu);
        q = warp_sum(q);
        const float inv = 1.f / sqrtf(q / float(C) + kLnEps);
        if (y) {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int c = 2 * (lane + 32 * j);
                const float2 g = ld2(gamma, c), b = ld2(beta, c);
                st2(y, r * C + c, make_float2(g.x * ((v[j].x - mu) * inv) + b.x, g.y * ((v[j].y - mu) * inv) + b.y));
            }
        }
        if (lane == 0 && stats) stats[r] = make_float2(mu, inv);
    }
}

// VJP: dx = inv (g*gamma - mean(g*gamma) - xh mean(g*gamma*xh)); dres_out = dres_in + dx
// (fp32, dres_in may alias dres_out), optional bf16 copy; dgamma/dbeta per-block partials
// [block][2C] (warps summed in a fixed order through shared memory).  A warp takes R rows per
// iteration and issues every load of them (stats, x, dy, dres_in) before the first reduction,
// so each iteration waits out one DRAM round trip instead of 2R.
template <int V>
constexpr int ln_bwd_rows() { return V <= 2 ? 4 : V <= 4 ? 2 : 1; }

template <int V, typename XT>
__global__ void __launch_bounds__(kRowWarps * 32)
    ln_bwd_kernel(const float* __restrict__ dy, const XT* __restrict__ x, const float2* __restrict__ stats,
                  const float* __restrict__ gamma, int64_t rows, const float* dres_in, float* dres_out,
                  __nv_bfloat16* __restrict__ dres_bf, float* __restrict__ part) {
    constexpr int C = 64 * V, R = ln_bwd_rows<V>();
    __shared__ float red[2 * C];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2 dg[V], db[V];
#pragma unroll
    for (int j = 0; j < V; ++j) dg[j] = db[j] = make_float2(0.f, 0.f);
    for (int64_t r0 = (int64_t(blockIdx.x) * kRowWarps + warp) * R; r0 < rows;
         r0 += int64_t(gridDim.x) * kRowWarps * R) {
        float2 st[R], xv[R][V], g[R][V], o[R][V];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int64_t r = r0 + q;
            if (r >= rows) break;
            st[q] = stats[r];
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int64_t i = r * C + 2 * (lane + 32 * j);
                xv[q][j] = ld2(x, i);
                g[q][j] = ld2(dy, i);
                o[q][j] = dres_in ? ld2(dres_in, i) : make_float2(0.f, 0.f);
            }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int64_t r = r0 + q;
            if (r >= rows) break;
            float s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const float2 ga = ld2(gamma, 2 * (lane + 32 * j));
                const float2 xh = make_float2((xv[q][j].x - st[q].x) * st[q].y, (xv[q][j].y - st[q].x) * st[q].y);
                const float2 gg = make_float2(g[q][j].x * ga.x, g[q][j].y * ga.y);
                s1 += gg.x + gg.y;
                s2 += gg.x * xh.x + gg.y * xh.y;
                dg[j].x += g[q][j].x * xh.x;
                dg[j].y += g[q][j].y * xh.y;
                db[j].x += g[q][j].x;
                db[j].y += g[q][j].y;
                xv[q][j] = xh;  // x-hat from here on
                g[q][j] = gg;   // g * gamma
            }
            s1 = warp_sum(s1);
            s2 = warp_sum(s2);
            const float m1 = s1 / float(C), m2 = s2 / float(C);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int64_t i = r * C + 2 * (lane + 32 * j);
                const float2 d = make_float2(st[q].y * (g[q][j].x - m1 - xv[q][j].x * m2) + o[q][j].x,
                                             st[q].y * (g[q][j].y - m1 - xv[q][j].y * m2) + o[q][j].y);
                if (dres_out) st2(dres_out, i, d);
                if (dres_bf) st2(dres_bf, i, d);
            }
        }
    }
    if (!part) return;
    for (int w = 0; w < kRowWarps; ++w) {
        if (warp == w) {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int c = 2 * (lane + 32 * j);
                if (w == 0) {
                    red[c] = dg[j].x;
                    red[c + 1] = dg[j].y;
                    red[C + c] = db[j].x;
                    red[C + c + 1] = db[j].y;
                } else {
                    red[c] += dg[j].x;
                    red[c + 1] += dg[j].y;
                    red[C + c] += db[j].x;
                    red[C + c + 1] += db[j].y;
                }
            }
        }
        __syncthreads();
    }
    for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) part[int64_t(blockIdx.x) * 2 * C + c] = red[c];
}

// out[c] += sum_p part[p * width + c]: one warp per column, lane-strided partial sums and a
// fixed butterfly (deterministic)
__global__ void colsum_partials_kernel(const float* __restrict__ part, int nparts, int width, float* __restrict__ out0,
                                       int split, float* __restrict__ out1) {
    const int lane = threadIdx.x & 31;
    for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < width; c += (gridDim.x * blockDim.x) >> 5) {
        float s = 0.f;
        for (int p = lane; p < nparts; p += 32) s += part[int64_t(p) * width + c];
        s = warp_sum(s);
        if (lane) continue;
        if (c < split) {
            if (out0) out0[c] += s;
        } else if (out1) {
            out1[c - split] += s;
        }
    }
}
static unsigned colsum_blocks(int64_t width) { return unsigned((width * 32 + 255) / 256); }

template <typename XT>
static int ln_fwd_t(const XT* x, const __nv_bfloat16* add, float* xo, __nv_bfloat16* xo_bf, const float* g,
                    const float* b, int64_t rows, int64_t C, __nv_bfloat16* y, float2* stats, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    // one row per warp: the rows of a wave are all in flight (a capped grid walking several rows
    // per warp kept the forward at ~28 % of DRAM throughput, 43 % warps active)
    const unsigned nb = row_blocks(rows, kRowWarps, 64 * kNumSMs);
    switch (C) {
#define AFFMAE_LNF(V_) \
    case 64 * V_: ln_fwd_kernel<V_, XT><<<nb, kRowWarps * 32, 0, st>>>(x, add, xo, xo_bf, g, b, rows, y, stats); break;
        AFFMAE_LNF(1)
        AFFMAE_LNF(2)
        AFFMAE_LNF(3)
        AFFMAE_LNF(4)
        AFFMAE_LNF(6)
        AFFMAE_LNF(8)
        AFFMAE_LNF(12)
        AFFMAE_LNF(16)
#undef AFFMAE_LNF
        default:
            return fail(AFFMAE_EUNSUPPORTED, "model layer_norm: width must be 64 * {1,2,3,4,6,8,12,16}");
    }
    AFFMAE_LAUNCH_CHECK("ln_fwd_kernel");
    return AFFMAE_OK;
}

int ln_fwd(const float* x, const __nv_bfloat16* add, float* xo, __nv_bfloat16* xo_bf, const float* g, const float* b,
           int64_t rows, int64_t C, __nv_bfloat16* y, float2* stats, cudaStream_t st) {
    return ln_fwd_t<float>(x, add, xo, xo_bf, g, b, rows, C, y, stats, st);
}
int ln_fwd_bf(const __nv_bfloat16* x, float* xo, const float* g, const float* b, int64_t rows, int64_t C,
              __nv_bfloat16* y, float2* stats, cudaStream_t st) {
    return ln_fwd_t<__nv_bfloat16>(x, nullptr, xo, nullptr, g, b, rows, C, y, stats, st);
}

// one iteration per warp while the grid stays under 4 blocks per SM
static int ln_bwd_rows_of(int64_t C) { return C <= 128 ? 4 : C <= 256 ? 2 : 1; }
unsigned ln_bwd_blocks(int64_t rows, int64_t C) { return row_blocks(rows, kRowWarps * ln_bwd_rows_of(C), 4 * kNumSMs); }

template <typename XT>
static int ln_bwd_t(const float* dy, const XT* x, const float2* stats, const float* g, int64_t rows, int64_t C,
                    const float* dres_in, float* dres_out, __nv_bfloat16* dres_bf, float* dgamma, float* dbeta,
                    float* part, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    const unsigned nb = ln_bwd_blocks(rows, C);
    float* pp = (dgamma || dbeta) ? part : nullptr;
    switch (C) {
#define AFFMAE_LNB(V_)                                                                                           \
    case 64 * V_:                                                                                                \
        ln_bwd_kernel<V_, XT><<<nb, kRowWarps * 32, 0, st>>>(dy, x, stats, g, rows, dres_in, dres_out, dres_bf, pp); \
        break;
        AFFMAE_LNB(1)
        AFFMAE_LNB(2)
        AFFMAE_LNB(3)
        AFFMAE_LNB(4)
        AFFMAE_LNB(6)
        AFFMAE_LNB(8)
        AFFMAE_LNB(12)
        AFFMAE_LNB(16)
#undef AFFMAE_LNB
        default:
            return fail(AFFMAE_EUNSUPPORTED, "model layer_norm: width must be 64 * {1,2,3,4,6,8,12,16}");
    }
    if (pp) colsum_partials_kernel<<<colsum_blocks(2 * C), 256, 0, st>>>(pp, int(nb), int(2 * C), dgamma,
                                                                                   int(C), dbeta);
    AFFMAE_LAUNCH_CHECK("ln_bwd_kernel");
    return AFFMAE_OK;
}

int ln_bwd(const float* dy, const float* x, const float2* stats, const float* g, int64_t rows, int64_t C,
           const float* dres_in, float* dres_out, __nv_bfloat16* dres_bf, float* dgamma, float* dbeta, float* part,
           cudaStream_t st) {
    return ln_bwd_t<float>(dy, x, stats, g, rows, C, dres_in, dres_out, dres_bf, dgamma, dbeta, part, st);
}
int ln_bwd_bf(const float* dy, const __nv_bfloat16* x, const float2* stats, const float* g, int64_t rows, int64_t C,
              const float* dres_in, float* dres_out, __nv_bfloat16* dres_bf, float* dgamma, float* dbeta, float* part,
              cudaStream_t st) {
    return ln_bwd_t<__nv_bfloat16>(dy, x, stats, g, rows, C, dres_in, dres_out, dres_bf, dgamma, dbeta, part, st);
}
size_t ln_bwd_part_floats(int64_t rows, int64_t C) { return size_t(ln_bwd_blocks(rows, C)) * 2 * size_t(C); }

// ------------------------------------------------------------ positional MLP
// hidden = GELU(c W1^T + b1), c = coords / image (scaled_coords, pipeline.cpp:48-52);
// W1 stored [16][2] (out, in).  H [rows, 16] bf16 feeds the second layer's GEMM.
__global__ void pos_hidden_fwd_kernel(const float2* __restrict__ coords, int64_t rows, float inv_image,
                                      const float* __restrict__ w1, const float* __restrict__ b1,
                                      __nv_bfloat16* __restrict__ h) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
        const float2 c = coords[r];
        const float cx = c.x * inv_image, cy = c.y * inv_image;
        alignas(16) __nv_bfloat162 o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float p0 = cx * w1[4 * j] + cy * w1[4 * j + 1] + b1[2 * j];
            const float p1 = cx * w1[4 * j + 2] + cy * w1[4 * j + 3] + b1[2 * j + 1];
            o[j] = __floats2bfloat162_rn(gelu_f(p0), gelu_f(p1));
        }
        uint4* dst = reinterpret_cast<uint4*>(h + r * 16);
        dst[0] = *reinterpret_cast<const uint4*>(&o[0]);
        dst[1] = *reinterpret_cast<const uint4*>(&o[4]);
    }
}

// dpre = dH * gelu'(pre); partials [block][48] = {dW1 [16][2], db1 [16]}
constexpr int kPosBlock = 256;
__global__ void __launch_bounds__(kPosBlock) pos_hidden_bwd_kernel(const float2* __restrict__ coords, int64_t rows,
                                                                    float inv_image, const float* __restrict__ w1,
                                                                    const float* __restrict__ b1,
                                                                    const float* __restrict__ dh,
                                                                    float* __restrict__ part) {
    __shared__ float red[kPosBlock / 32][48];
    float acc[48];
#pragma unroll
    for (int i = 0; i < 48; ++i) acc[i] = 0.f;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
        const float2 c = coords[r];
        const float cx = c.x * inv_image, cy = c.y * inv_image;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float pre = cx * w1[2 * j] + cy * w1[2 * j + 1] + b1[j];
            const float d = dh[r * 16 + j] * gelu_grad_f(pre);
            acc[2 * j] += d * cx;
            acc[2 * j + 1] += d * cy;
            acc[32 + j] += d;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 48; ++i) {
        const float s = warp_sum(acc[i]);
        if (lane == 0) red[warp][i] = s;
    }
    __syncthreads();
    if (threadIdx.x < 48) {
        float s = 0.f;
        for (int w = 0; w < kPosBlock / 32; ++w) s += red[w][threadIdx.x];
        part[int64_t(blockIdx.x) * 48 + threadIdx.x] = s;
    }
}

int pos_hidden_fwd(const float* coords, int64_t rows, float inv_image, const float* w1, const float* b1,
                   __nv_bfloat16* h, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    pos_hidden_fwd_kernel<<<row_blocks(rows, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(coords), rows,
                                                                  inv_image, w1, b1, h);
    AFFMAE_LAUNCH_CHECK("pos_hidden_fwd_kernel");
    return AFFMAE_OK;
}
unsigned pos_bwd_blocks(int64_t rows) { return row_blocks(rows, kPosBlock * 4, kNumSMs); }
int pos_hidden_bwd(const float* coords, int64_t rows, float inv_image, const float* w1, const float* b1,
                   const float* dh, float* dw1, float* db1, float* part, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    const unsigned nb = pos_bwd_blocks(rows);
    pos_hidden_bwd_kernel<<<nb, kPosBlock, 0, st>>>(reinterpret_cast<const float2*>(coords), rows, inv_image, w1, b1,
                                                    dh, part);
    colsum_partials_kernel<<<colsum_blocks(48), 256, 0, st>>>(part, int(nb), 48, dw1, 32, db1);
    AFFMAE_LAUNCH_CHECK("pos_hidden_bwd_kernel");
    return AFFMAE_OK;
}

// ------------------------------------------------------------------- scorer
// scores = sigmoid(hid . w2 + b2), hid [rows, 16] bf16 (GELU output of the first GEMM)
__global__ void scorer_out_fwd_kernel(const __nv_bfloat16* __restrict__ hid, int64_t rows, const float* __restrict__ w2,
                                      const float* __restrict__ b2, float* __restrict__ scores) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
        float z = 0.f;
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
            const float2 h = ld2(hid, r * 16 + j);
            z += h.x * w2[j] + h.y * w2[j + 1];
        }
        z += b2[0];
        scores[r] = float(1.0 / (1.0 + exp(-double(z))));
    }
}

// dz = ds s (1 - s); dhid = dz w2 (bf16); partials [block][17] = {dw2 [16], db2}
__global__ void __launch_bounds__(kPosBlock) scorer_out_bwd_kernel(const __nv_bfloat16* __restrict__ hid,
                                                                    const float* __restrict__ scores,
                                                                    const float* __restrict__ dscores, int64_t rows,
                                                                    const float* __restrict__ w2,
                                                                    __nv_bfloat16* __restrict__ dhid,
                                                                    float* __restrict__ part) {
    __shared__ float red[kPosBlock / 32][17];
    float acc[17];
#pragma unroll
    for (int i = 0; i < 17; ++i) acc[i] = 0.f;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
        const float s = scores[r];
        const float dz = dscores[r] * s * (1.f - s);
        alignas(16) __nv_bfloat162 o[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
            const float2 h = ld2(hid, r * 16 + j);
            acc[j] += dz * h.x;
            acc[j + 1] += dz * h.y;
            o[j / 2] = __floats2bfloat162_rn(dz * w2[j], dz * w2[j + 1]);
        }
        acc[16] += dz;
        uint4* dst = reinterpret_cast<uint4*>(dhid + r * 16);
        dst[0] = *reinterpret_cast<const uint4*>(&o[0]);
        dst[1] = *reinterpret_cast<const uint4*>(&o[4]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 17; ++i) {
        const float s = warp_sum(acc[i]);
        if (lane == 0) red[warp][i] = s;
    }
    __syncthreads();
    if (threadIdx.x < 17) {
        float s = 0.f;
        for (int w = 0; w < kPosBlock / 32; ++w) s += red[w][threadIdx.x];
        part[int64_t(blockIdx.x) * 17 + threadIdx.x] = s;
    }
}

int scorer_out_fwd(const __nv_bfloat16* hid, int64_t rows, const float* w2, const float* b2, float* scores,
                   cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    scorer_out_fwd_kernel<<<row_blocks(rows, 256), 256, 0, st>>>(hid, rows, w2, b2, scores);
    AFFMAE_LAUNCH_CHECK("scorer_out_fwd_kernel");
    return AFFMAE_OK;
}
int scorer_out_bwd(const __nv_bfloat16* hid, const float* scores, const float* dscores, int64_t rows, const float* w2,
                   __nv_bfloat16* dhid, float* dw2, float* db2, float* part, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    const unsigned nb = pos_bwd_blocks(rows);
    scorer_out_bwd_kernel<<<nb, kPosBlock, 0, st>>>(hid, scores, dscores, rows, w2, dhid, part);
    colsum_partials_kernel<<<colsum_blocks(17), 256, 0, st>>>(part, int(nb), 17, dw2, 16, db2);
    AFFMAE_LAUNCH_CHECK("scorer_out_bwd_kernel");
    return AFFMAE_OK;
}

// ------------------------------------------------------ decoder offset head
// pre = fq W^T + b (W stored [2][dd]); off = NormClamp(pre, limit); qpos = refs + off
template <int V>
__global__ void __launch_bounds__(kRowWarps * 32)
    offset_fwd_kernel(const float* __restrict__ fq, int64_t rows, const float* __restrict__ w,
                      const float* __restrict__ b, double limit, const float2* __restrict__ refs,
                      float2* __restrict__ pre, float2* __restrict__ qpos) {
    constexpr int C = 64 * V;
    const int lane = threadIdx.x & 31;
    for (int64_t r = int64_t(blockIdx.x) * kRowWarps + (threadIdx.x >> 5); r < rows;
         r += int64_t(gridDim.x) * kRowWarps) {
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int c = 2 * (lane + 32 * j);
            const float2 x = ld2(fq, r * C + c), w0 = ld2(w, c), w1 = ld2(w, C + c);
            s0 += x.x * w0.x + x.y * w0.y;
            s1 += x.x * w1.x + x.y * w1.y;
        }
        s0 = warp_sum(s0) + b[0];
        s1 = warp_sum(s1) + b[1];
        if (lane == 0) {
            pre[r] = make_float2(s0, s1);
            const double rr = sqrt(double(s0) * double(s0) + double(s1) * double(s1));
            const double f = rr > limit ? limit / rr : 1.0;
            const float o0 = float(double(s0) * f), o1 = float(double(s1) * f);
            const float2 q = refs[r];
            qpos[r] = make_float2(q.x + o0, q.y + o1);
        }
    }
}

// NormClampOp::backward (pipeline.cpp:104-125) then the linear's VJP:
// dfq += dpre W (in place), partials [block][2C + 2] = {dW [2][C], db [2]}
template <int V>
__global__ void __launch_bounds__(kRowWarps * 32)
    offset_bwd_kernel(const float* __restrict__ fq, int64_t rows, const float* __restrict__ w, double limit,
                      const float2* __restrict__ pre, const float2* __restrict__ dqpos, float* __restrict__ dfq,
                      float* __restrict__ part) {
    constexpr int C = 64 * V;
    __shared__ float red[2 * C + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2 a0[V], a1[V];
    float g0 = 0.f, g1 = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) a0[j] = a1[j] = make_float2(0.f, 0.f);
    // R rows per warp iteration: their loads are independent (memory-level parallelism)
    constexpr int R = 4;
    const int64_t step = int64_t(gridDim.x) * kRowWarps * R;
    for (int64_t r0 = (int64_t(blockIdx.x) * kRowWarps + warp) * R; r0 < rows; r0 += step) {
        float d0[R], d1[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            d0[i] = d1[i] = 0.f;
            const int64_t r = r0 + i;
            if (r >= rows) continue;
            const float2 p = pre[r], g = dqpos[r];
            const double rr = sqrt(double(p.x) * double(p.x) + double(p.y) * double(p.y));
            d0[i] = g.x;
            d1[i] = g.y;
            if (rr > limit) {
                const double f = limit / rr;
                const double dot = (double(g.x) * p.x + double(g.y) * p.y) / (rr * rr);
                d0[i] = float(f * (g.x - dot * p.x));
                d1[i] = float(f * (g.y - dot * p.y));
            }
            g0 += d0[i];
            g1 += d1[i];
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int c = 2 * (lane + 32 * j);
            const float2 w0 = ld2(w, c), w1 = ld2(w, C + c);
            float2 x[R], o[R];
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (r0 + i < rows) {
                    x[i] = ld2(fq, (r0 + i) * C + c);
                    o[i] = ld2(dfq, (r0 + i) * C + c);
                }
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (r0 + i < rows) {
                    a0[j].x += d0[i] * x[i].x;
                    a0[j].y += d0[i] * x[i].y;
                    a1[j].x += d1[i] * x[i].x;
                    a1[j].y += d1[i] * x[i].y;
                    o[i].x += d0[i] * w0.x + d1[i] * w1.x;
                    o[i].y += d0[i] * w0.y + d1[i] * w1.y;
                    st2(dfq, (r0 + i) * C + c, o[i]);
                }
        }
    }
    for (int ww = 0; ww < kRowWarps; ++ww) {
        if (warp == ww) {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int c = 2 * (lane + 32 * j);
                const float v[4] = {a0[j].x, a0[j].y, a1[j].x, a1[j].y};
                const int at[4] = {c, c + 1, C + c, C + c + 1};
#pragma unroll
                for (int e = 0; e < 4; ++e) red[at[e]] = (ww == 0 ? 0.f : red[at[e]]) + v[e];
            }
            if (lane == 0) {
                red[2 * C] = (ww == 0 ? 0.f : red[2 * C]) + g0;
                red[2 * C + 1] = (ww == 0 ? 0.f : red[2 * C + 1]) + g1;
            }
        }
        __syncthreads();
    }
    for (int c = threadIdx.x; c < 2 * C + 2; c += blockDim.x) part[int64_t(blockIdx.x) * (2 * C + 2) + c] = red[c];
}

int offset_fwd(const float* fq, int64_t rows, int64_t C, const float* w, const float* b, double limit,
               const float* refs, float* pre, float* qpos, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    const unsigned nb = row_blocks(rows, kRowWarps);
    const auto* r2 = reinterpret_cast<const float2*>(refs);
    auto* p2 = reinterpret_cast<float2*>(pre);
    auto* q2 = reinterpret_cast<float2*>(qpos);
    switch (C) {
#define AFFMAE_OFF(V_) \
    case 64 * V_: offset_fwd_kernel<V_><<<nb, kRowWarps * 32, 0, st>>>(fq, rows, w, b, limit, r2, p2, q2); break;
        AFFMAE_OFF(1)
        AFFMAE_OFF(2)
        AFFMAE_OFF(4)
        AFFMAE_OFF(8)
        AFFMAE_OFF(16)
#undef AFFMAE_OFF
        default:
            return fail(AFFMAE_EUNSUPPORTED, "decoder offset head: width must be 64, 128, 256, 512 or 1024");
    }
    AFFMAE_LAUNCH_CHECK("offset_fwd_kernel");
    return AFFMAE_OK;
}
unsigned offset_bwd_blocks(int64_t rows) { return row_blocks(rows, 4 * kRowWarps, 4 * kNumSMs); }
int offset_bwd(const float* fq, int64_t rows, int64_t C, const float* w, double limit, const float* pre,
               const float* dqpos, float* dfq, float* dw, float* db, float* part, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    const unsigned nb = offset_bwd_blocks(rows);
    const auto* p2 = reinterpret_cast<const float2*>(pre);
    const auto* d2 = reinterpret_cast<const float2*>(dqpos);
    switch (C) {
#define AFFMAE_OFFB(V_)                                                                                   \
    case 64 * V_: offset_bwd_kernel<V_><<<nb, kRowWarps * 32, 0, st>>>(fq, rows, w, limit, p2, d2, dfq, part); \
        break;
        AFFMAE_OFFB(1)
        AFFMAE_OFFB(2)
        AFFMAE_OFFB(4)
        AFFMAE_OFFB(8)
        AFFMAE_OFFB(16)
#undef AFFMAE_OFFB
        default:
            return fail(AFFMAE_EUNSUPPORTED, "decoder offset head: width must be 64, 128, 256, 512 or 1024");
    }
    colsum_partials_kernel<<<colsum_blocks(2 * C + 2), 256, 0, st>>>(part, int(nb), int(2 * C + 2), dw,
                                                                             int(2 * C), db);
    AFFMAE_LAUNCH_CHECK("offset_bwd_kernel");
    return AFFMAE_OK;
}

// ------------------------------------------------------------ gathers, masks
// Cells of each image whose mask byte == want, ascending: global rows b*cells + cell and
// pixel centres (c*patch + patch/2, r*patch + patch/2) (grid_points, geometry.cpp:44-50;
// visible / masked lists of Model::encode / decode, pipeline.cpp:412-427, 481-492).
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) cell_rows_kernel(const uint8_t* __restrict__ masked, int64_t gw,
                                                                 int64_t cells, int want, int64_t n, double patch,
                                                                 int32_t* __restrict__ rows,
                                                                 float2* __restrict__ coords) {
    __shared__ int32_t wsum[32];
    const uint8_t* m = masked + int64_t(blockIdx.x) * cells;
    const int64_t per = (cells + kScanThreads - 1) / kScanThreads;
    const int64_t lo = threadIdx.x * per, hi = lo + per < cells ? lo + per : cells;
    int32_t cnt = 0;
    for (int64_t i = lo; i < hi; ++i) cnt += (m[i] != 0) == (want != 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    int64_t pos = inc - cnt + (warp > 0 ? wsum[warp - 1] : 0);
    for (int64_t i = lo; i < hi; ++i)
        if ((m[i] != 0) == (want != 0)) {
            if (pos < n) {
                const int64_t o = int64_t(blockIdx.x) * n + pos;
                if (rows) rows[o] = int32_t(int64_t(blockIdx.x) * cells + i);
                if (coords) {
                    const int64_t rr = i / gw, cc = i - rr * gw;
                    coords[o] = make_float2(float(double(cc) * patch + patch * 0.5),
                                            float(double(rr) * patch + patch * 0.5));
                }
            }
            ++pos;
        }
}

int cell_rows(const uint8_t* masked, int64_t batch, int64_t gh, int64_t gw, int want, int64_t n, double patch,
              int32_t* rows, float* coords, cudaStream_t st) {
    if (batch <= 0) return AFFMAE_OK;
    cell_rows_kernel<<<unsigned(batch), kScanThreads, 0, st>>>(masked, gw, gh * gw, want, n, patch, rows,
                                                               reinterpret_cast<float2*>(coords));
    AFFMAE_LAUNCH_CHECK("cell_rows_kernel");
    return AFFMAE_OK;
}

// out[r] = bf16(patches[rows[r]])  (p2 columns, 8 per thread)
__global__ void gather_rows_bf16_kernel(const float* __restrict__ src, const int32_t* __restrict__ rows, int64_t n,
                                        int64_t p2, __nv_bfloat16* __restrict__ out) {
    const int64_t per = p2 / 8;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n * per; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = t / per, e = (t - r * per) * 8;
        const float* s = src + int64_t(rows[r]) * p2 + e;
        const float4 a = *reinterpret_cast<const float4*>(s), b = *reinterpret_cast<const float4*>(s + 4);
        alignas(16) __nv_bfloat162 o[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
        *reinterpret_cast<uint4*>(out + r * p2 + e) = *reinterpret_cast<const uint4*>(o);
    }
}
int gather_rows_bf16(const float* src, const int32_t* rows, int64_t n, int64_t p2, __nv_bfloat16* out, cudaStream_t st) {
    if (n <= 0) return AFFMAE_OK;
    if (p2 % 8) return fail(AFFMAE_EUNSUPPORTED, "gather_rows: width must be a multiple of 8");
    gather_rows_bf16_kernel<<<row_blocks(n * p2 / 8, 256, 16 * kNumSMs), 256, 0, st>>>(src, rows, n, p2, out);
    AFFMAE_LAUNCH_CHECK("gather_rows_bf16_kernel");
    return AFFMAE_OK;
}

// next-stage coordinates: out[b, r] = coords[b, retained[b, r]] (pipeline.cpp:459-464)
__global__ void gather_coords_kernel(const float2* __restrict__ coords, const int32_t* __restrict__ ret, int64_t batch,
                                     int64_t n, int64_t r, float2* __restrict__ out) {
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < batch * r; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / r;
        out[t] = coords[b * n + ret[t]];
    }
}
int gather_coords(const float* coords, const int32_t* ret, int64_t batch, int64_t n, int64_t r, float* out,
                  cudaStream_t st) {
    if (batch * r <= 0) return AFFMAE_OK;
    gather_coords_kernel<<<row_blocks(batch * r, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(coords), ret,
                                                                      batch, n, r, reinterpret_cast<float2*>(out));
    AFFMAE_LAUNCH_CHECK("gather_coords_kernel");
    return AFFMAE_OK;
}

// ------------------------------------------------------------- elementwise
// out = a + b (fp32 + bf16 -> fp32, optional bf16 copy); a may be null (then out = b) or
// a row vector broadcast over rows (a_row != 0: the decoder's repeated mask token)
__global__ void add_f32_bf16_kernel(const float* __restrict__ a, int a_row, const __nv_bfloat16* __restrict__ b,
                                    int64_t rows, int64_t cols, float* __restrict__ out,
                                    __nv_bfloat16* __restrict__ out_bf) {
    const int64_t n2 = rows * cols / 2;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n2; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = 2 * t;
        float2 v = ld2(b, i);
        if (a) {
            const float2 x = ld2(a, a_row ? i % cols : i);
            v.x += x.x;
            v.y += x.y;
        }
        if (out) st2(out, i, v);
        if (out_bf) st2(out_bf, i, v);
    }
}
int add_f32_bf16(const float* a, int a_row, const __nv_bfloat16* b, int64_t rows, int64_t cols, float* out,
                 __nv_bfloat16* out_bf, cudaStream_t st) {
    if (rows * cols <= 0) return AFFMAE_OK;
    add_f32_bf16_kernel<<<row_blocks(rows * cols / 2, 256, 16 * kNumSMs), 256, 0, st>>>(a, a_row, b, rows, cols, out,
                                                                                        out_bf);
    AFFMAE_LAUNCH_CHECK("add_f32_bf16_kernel");
    return AFFMAE_OK;
}

// y = GELU_erf(pre) (gelu_fwd, src/tape.cpp:104-107), 8 bf16 per thread: the MLP's first GEMM
// stores the pre-activation (its backward needs it) and this pass applies the activation --
// faster than the GEMM's fused GELU epilogue at the model's shapes (0.24 -> 0.06 + 0.07 ms
// for 196608 x 512, tools/decoder_probe.py)
__global__ void gelu_fwd_kernel(const uint4* __restrict__ pre, int64_t n8, uint4* __restrict__ y) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
        const uint4 p = pre[i];
        const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&p);
        uint4 o;
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 x = __bfloat1622float2(ph[j]);
            oh[j] = __floats2bfloat162_rn(gelu_f(x.x), gelu_f(x.y));
        }
        y[i] = o;
    }
}
int gelu_fwd(const bf16* pre, int64_t n, bf16* y, cudaStream_t st) {
    if (n <= 0) return AFFMAE_OK;
    if (n % 8) return fail(AFFMAE_EUNSUPPORTED, "gelu_fwd: element count must be a multiple of 8");
    gelu_fwd_kernel<<<row_blocks(n / 8, 256, 16 * kNumSMs), 256, 0, st>>>(reinterpret_cast<const uint4*>(pre), n / 8,
                                                                         reinterpret_cast<uint4*>(y));
    AFFMAE_LAUNCH_CHECK("gelu_fwd_kernel");
    return AFFMAE_OK;
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ y) {
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; 2 * t < n; t += int64_t(gridDim.x) * blockDim.x)
        st2(y, 2 * t, ld2(x, 2 * t));
}
int cast_bf16(const float* x, int64_t n, __nv_bfloat16* y, cudaStream_t st) {
    if (n <= 0) return AFFMAE_OK;
    if (n % 2) return fail(AFFMAE_EUNSUPPORTED, "cast_bf16: even element count required");
    cast_bf16_kernel<<<row_blocks(n / 2, 256, 16 * kNumSMs), 256, 0, st>>>(x, n, y);
    AFFMAE_LAUNCH_CHECK("cast_bf16_kernel");
    return AFFMAE_OK;
}

// dense fp32 [rows, cols] -> bf16 rows of stride ldy (a column slice of a wider matrix)
// four columns per thread (16-byte loads, 8-byte stores); blockIdx.y walks the 4-column groups
// of a row block, so no per-element 64-bit division
__global__ void cast_bf16_2d_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, __nv_bfloat16* __restrict__ y,
                                    int64_t ldy) {
    const int64_t q4 = cols / 4;
    for (int64_t r = int64_t(blockIdx.x) * (blockDim.x / q4) + threadIdx.x / q4; r < rows;
         r += int64_t(gridDim.x) * (blockDim.x / q4)) {
        const int64_t c = 4 * (threadIdx.x % q4);
        const float4 v = *reinterpret_cast<const float4*>(x + r * cols + c);
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 o;
        o.x = *reinterpret_cast<const uint32_t*>(&lo);
        o.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(y + r * ldy + c) = o;
    }
}
int cast_bf16_2d(const float* x, int64_t rows, int64_t cols, __nv_bfloat16* y, int64_t ldy, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    if (cols % 4 || ldy % 4 || cols / 4 > 256) return fail(AFFMAE_EUNSUPPORTED, "cast_bf16_2d: width");
    const int64_t per = 256 / (cols / 4);  // rows per 256-thread block
    cast_bf16_2d_kernel<<<row_blocks(rows, int(per), 16 * kNumSMs), unsigned(per * (cols / 4)), 0, st>>>(
        x, rows, cols, y, ldy);
    AFFMAE_LAUNCH_CHECK("cast_bf16_2d_kernel");
    return AFFMAE_OK;
}

// column sums of an fp32 [rows, cols] matrix into out (+=): per-block partials + fixed-order sum
__global__ void colsum_f32_partial_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t rows_per,
                                          float* __restrict__ part) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    const int64_t r0 = int64_t(blockIdx.y) * rows_per, r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;  // four independent loads in flight
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4) {
        s0 += x[r * cols + c];
        s1 += x[(r + 1) * cols + c];
        s2 += x[(r + 2) * cols + c];
        s3 += x[(r + 3) * cols + c];
    }
    for (; r < r1; ++r) s0 += x[r * cols + c];
    part[int64_t(blockIdx.y) * cols + c] = (s0 + s1) + (s2 + s3);
}
constexpr int kColChunks = 1024;  // row chunks: enough blocks to fill the GPU for narrow rows
int colsum_f32(const float* x, int64_t rows, int64_t cols, float* out, float* part, cudaStream_t st) {
    if (rows <= 0) return AFFMAE_OK;
    const int64_t rows_per = (rows + kColChunks - 1) / kColChunks;
    colsum_f32_partial_kernel<<<dim3(unsigned((cols + 255) / 256), kColChunks), 256, 0, st>>>(x, rows, cols, rows_per,
                                                                                           part);
    colsum_partials_kernel<<<colsum_blocks(cols), 256, 0, st>>>(part, kColChunks, int(cols), out, int(cols),
                                                                          nullptr);
    AFFMAE_LAUNCH_CHECK("colsum_f32");
    return AFFMAE_OK;
}
size_t colsum_part_floats(int64_t cols) { return size_t(kColChunks) * size_t(cols); }

// bf16 shadow of the GEMM-operand parameters (the first n values of the fp32 arena)
int shadow_cast(const float* p, int64_t n, __nv_bfloat16* pb, cudaStream_t st) { return cast_bf16(p, n, pb, st); }

}  // namespace mk
}  // namespace affmae_b200
