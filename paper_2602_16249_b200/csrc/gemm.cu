// Dense linear layers of the training step on the hand-written tcgen05 GEMM (gemm_tc.cu):
// the reference Tape's matmul + bias (+ gelu_erf) (proj/src/tape.cpp:24-114,
// proj/src/pipeline.cpp:388-400,453-458) and their VJPs.
//   linear_fwd           y = act(x W^T + b)                x [M, K], W [N, K] (nn.Linear layout)
//   linear_fwd_gelu_aux  pre = x W^T + b, y = GELU(pre)    one pass, both stored
//   linear_fwd_add       y = x W^T + b + c                 residual added before the rounding
//   linear_bwd           dX = dY W (bf16), dW += dY^T X (fp32, split-K partials reduced in a
//                        fixed order), db += column sums of dY (fixed order)
//   linear_dx_gelu       dH = (dY W) · GELU'(pre)          the MLP's fc2 input gradient with
//                        the activation's derivative fused (no dX round trip through HBM)
//   linear_dx_f32        dX = dY W + beta · dX             fp32 residual-stream gradients
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace affmae_b200 {

// cs_out: the weight-gradient form (A = dY read M-major) also sums dY's columns -- the bias
// gradient -- from its operand ring: cs_accum ? cs_out[m] += : cs_out[split * M + m] =
int tc_gemm(const void* a, bool a_mn, const void* b, bool b_mn, int64_t M, int64_t N, int64_t K, int epi,
            const float* bias, const void* aux, void* out, void* out2, float beta, int64_t ldo, int splits,
            cudaStream_t st, float* cs_out = nullptr, int cs_accum = 0);
int tc_gemm_pick_splits(int64_t M, int64_t N, int64_t K);

namespace {

enum { kStore = 0, kGeluAux = 1, kAdd = 2, kGeluBwd = 3, kF32 = 4, kGelu = 5 };

// dpre = dy * gelu'(pre), gelu'(x) = Phi(x) + x phi(x)  (tape.cpp gelu_bwd), 8 bf16 per thread
__global__ void gelu_bwd_kernel(const uint4* __restrict__ pre, const uint4* __restrict__ dy, int64_t n8,
                                uint4* __restrict__ dpre) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
        const uint4 p = __ldg(pre + i), g = __ldg(dy + i);
        const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&p);
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&g);
        uint4 o;
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 x2 = __bfloat1622float2(ph[j]), g2 = __bfloat1622float2(gh[j]);
            float r[2];
            const float xs[2] = {x2.x, x2.y}, gs[2] = {g2.x, g2.y};
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float x = xs[e];
                const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
                const float pdf = 0.39894228040143268f * __expf(-0.5f * x * x);
                r[e] = gs[e] * (cdf + x * pdf);
            }
            oh[j] = __floats2bfloat162_rn(r[0], r[1]);
        }
        dpre[i] = o;
    }
}

// db[n] += sum_m dY[m, n] in two deterministic passes.  Pass 1: block b sums the rows of its
// chunk; a thread owns 8 consecutive columns (16-byte loads) and every (256 / groups)-th row
// of the chunk, four rows in flight; the row lanes are then added in lane order through shared
// memory.  Pass 2: one warp per column adds the chunk partials in a fixed order.
constexpr int kColsumThreads = 256;
__global__ void __launch_bounds__(kColsumThreads)
    colsum_partial_kernel(const __nv_bfloat16* __restrict__ dy, int64_t m, int64_t n, int64_t rows_per,
                          float* __restrict__ part) {
    extern __shared__ float red[];  // [lanes][8 * groups]
    const int64_t g8 = n / 8;
    const int groups = int(g8 < kColsumThreads ? g8 : kColsumThreads);
    const int lanes = kColsumThreads / groups;
    const int t = threadIdx.x;
    const int gi = t % groups, li = t / groups;
    const int64_t r0 = int64_t(blockIdx.x) * rows_per, r1 = r0 + rows_per < m ? r0 + rows_per : m;
    for (int64_t gbase = 0; gbase < g8; gbase += groups) {
        const int64_t g = gbase + gi;
        float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (li < lanes && g < g8) {
            const uint4* src = reinterpret_cast<const uint4*>(dy) + g;
            int64_t r = r0 + li;
#pragma unroll 1
            for (; r + 3 * lanes < r1; r += 4 * lanes) {
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(src + (r + int64_t(u) * lanes) * g8);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __bfloat1622float2(h[e]);
                        s[2 * e] += f.x;
                        s[2 * e + 1] += f.y;
                    }
                }
            }
            for (; r < r1; r += lanes) {
                const uint4 v = __ldg(src + r * g8);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(h[e]);
                    s[2 * e] += f.x;
                    s[2 * e + 1] += f.y;
                }
            }
        }
        if (li < lanes) {
#pragma unroll
            for (int e = 0; e < 8; ++e) red[li * 8 * groups + 8 * gi + e] = s[e];
        }
        __syncthreads();
        for (int c = t; c < 8 * groups; c += kColsumThreads) {
            const int64_t col = gbase * 8 + c;
            if (col >= n) continue;
            float a = 0.f;
            for (int l = 0; l < lanes; ++l) a += red[l * 8 * groups + c];
            part[int64_t(blockIdx.x) * n + col] = a;
        }
        __syncthreads();
    }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int64_t n, int chunks, float* __restrict__ db) {
    const int64_t col = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (col >= n) return;
    float s = 0.f;
    for (int c = lane; c < chunks; c += 32) s += part[int64_t(c) * n + col];
    s = warp_sum(s);
    if (lane == 0) db[col] += s;
}
constexpr int kColsumChunks = 2 * kNumSMs;

// dW += sum_l part[l]: a block owns 32 float4 columns; its 8 warps each sum the parts
// w, w + 8, ... of one column per lane (independent loads in flight), then warp 0 adds the 8
// warp sums in warp order -- a fixed order, so the result is deterministic
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float4* __restrict__ part, int64_t n4, int parts,
                                                            float4* __restrict__ dw) {
    __shared__ float4 red[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = int64_t(blockIdx.x) * 32; base < n4; base += int64_t(gridDim.x) * 32) {
        const int64_t i = base + lane;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n4) {
#pragma unroll 4
            for (int l = wid; l < parts; l += 8) {
                const float4 p = __ldg(part + int64_t(l) * n4 + i);
                s.x += p.x;
                s.y += p.y;
                s.z += p.z;
                s.w += p.w;
            }
        }
        red[wid][lane] = s;
        __syncthreads();
        if (wid == 0 && i < n4) {
            float4 o = dw[i];
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                o.x += red[w][lane].x;
                o.y += red[w][lane].y;
                o.z += red[w][lane].z;
                o.w += red[w][lane].w;
            }
            dw[i] = o;
        }
        __syncthreads();
    }
}

int check_shape(int64_t m, int64_t n, int64_t k, const char* what) {
    if (m < 1 || n < 1 || k < 1 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX)
        return fail(AFFMAE_ECONFIG, std::string(what) + ": bad shape");
    if (k % 8 || n % 8) return fail(AFFMAE_EUNSUPPORTED, std::string(what) + ": N and K must be multiples of 8");
    return AFFMAE_OK;
}

size_t colsum_bytes(int64_t n) { return size_t(kColsumChunks) * size_t(n) * 4 + 256; }
// dW [n, k] = dY^T X over m tokens, split into `splits` token ranges
size_t splitk_bytes(int64_t m, int64_t n, int64_t k) {
    const int s = tc_gemm_pick_splits(n, k, m);
    return s > 1 ? size_t(s) * size_t(n) * size_t(k) * 4 + 256 : 0;
}
float* align256(void* p) { return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255)); }

}  // namespace

// the forward needs no scratch (tensor maps travel as kernel parameters); kept in the ABI
size_t linear_workspace(int64_t, int64_t, int64_t) { return 256; }
size_t linear_bwd_workspace(int64_t m, int64_t n, int64_t k) { return colsum_bytes(n) + splitk_bytes(m, n, k); }

int linear_fwd(const void* x, const void* w, const float* bias, int64_t m, int64_t n, int64_t k, int act, void* y,
               void* ws, size_t ws_bytes, void* stream) {
    if (!x || !w || !bias || !y) return fail(AFFMAE_ECONFIG, "linear: null pointer");
    if (int rc = check_shape(m, n, k, "linear")) return rc;
    if (act == 0) return tc_gemm(x, false, w, false, m, n, k, kStore, bias, nullptr, y, nullptr, 0.f, n, 1, as_stream(stream));
    if (act == 1) return tc_gemm(x, false, w, false, m, n, k, kGelu, bias, nullptr, y, nullptr, 0.f, n, 1, as_stream(stream));
    return fail(AFFMAE_EUNSUPPORTED, "linear: act must be 0 (identity) or 1 (GELU)");
}

int linear_fwd_gelu_aux(const void* x, const void* w, const float* bias, int64_t m, int64_t n, int64_t k, void* y,
                        void* pre, void* ws, size_t ws_bytes, void* stream) {
    if (!x || !w || !bias || !y || !pre) return fail(AFFMAE_ECONFIG, "linear: null pointer");
    if (int rc = check_shape(m, n, k, "linear")) return rc;
    return tc_gemm(x, false, w, false, m, n, k, kGeluAux, bias, nullptr, pre, y, 0.f, n, 1, as_stream(stream));
}

int linear_fwd_add(const void* x, const void* w, const float* bias, int64_t m, int64_t n, int64_t k, const void* c,
                   void* y, void* ws, size_t ws_bytes, void* stream) {
    if (!x || !w || !bias || !y || !c) return fail(AFFMAE_ECONFIG, "linear: null pointer");
    if (int rc = check_shape(m, n, k, "linear")) return rc;
    return tc_gemm(x, false, w, false, m, n, k, kAdd, bias, c, y, nullptr, 0.f, n, 1, as_stream(stream));
}

int linear_dx_f32(const void* dy, const void* w, int64_t m, int64_t n, int64_t k, float* dx, float beta, void* ws,
                  size_t ws_bytes, void* stream) {
    if (!dy || !w || !dx) return fail(AFFMAE_ECONFIG, "linear dx: null pointer");
    if (int rc = check_shape(m, n, k, "linear dx")) return rc;
    return tc_gemm(dy, false, w, true, m, k, n, kF32, nullptr, nullptr, dx, nullptr, beta, k, 1, as_stream(stream));
}

int linear_dx_gelu(const void* dy, const void* w, const void* pre, int64_t m, int64_t n, int64_t k, void* dh,
                   void* stream) {
    if (!dy || !w || !pre || !dh) return fail(AFFMAE_ECONFIG, "linear dx gelu: null pointer");
    if (int rc = check_shape(m, n, k, "linear dx gelu")) return rc;
    return tc_gemm(dy, false, w, true, m, k, n, kGeluBwd, nullptr, pre, dh, nullptr, 0.f, k, 1, as_stream(stream));
}

int linear_bwd(const void* x, const void* w, const void* dy, int64_t m, int64_t n, int64_t k, void* dx, float* dw,
               float* db, void* ws, size_t ws_bytes, void* stream) {
    if (!x || !w || !dy) return fail(AFFMAE_ECONFIG, "linear bwd: null pointer");
    if (int rc = check_shape(m, n, k, "linear bwd")) return rc;
    if (ws_bytes < linear_bwd_workspace(m, n, k)) return fail(AFFMAE_ECONFIG, "linear bwd: workspace too small");
    cudaStream_t st = as_stream(stream);
    float* part = align256(ws);
    float* skpart = align256(reinterpret_cast<char*>(ws) + colsum_bytes(n));
    int rc = AFFMAE_OK;
    bool fused_db = false;
    // dX [m, k] = dY [m, n] · W [n, k]   (B read N-major from W's rows)
    if (dx && (rc = tc_gemm(dy, false, w, true, m, k, n, kStore, nullptr, nullptr, dx, nullptr, 0.f, k, 1, st)))
        return rc;
    if (dw) {
        // dW [n, k] += dY^T · X: A = dY read M-major, B = X read N-major, K = tokens; the same
        // GEMM sums dY's columns into db (per split, then a fixed-order sum over the splits)
        const int splits = tc_gemm_pick_splits(n, k, m);
        // the fused column sums pay where the weight gradient is split >= 8 ways (few output
        // tiles, HBM-bound main loop); a weight gradient with many tiles keeps its main loop on
        // the tensor pipe and takes the separate column-sum pass (profiles/r02l_gemm_probe.jsonl)
        fused_db = db && splits >= 8;
        if (splits < 2) {
            if ((rc = tc_gemm(dy, true, x, true, n, k, m, kF32, nullptr, nullptr, dw, nullptr, 1.f, k, 1, st)))
                return rc;
        } else {
            if ((rc = tc_gemm(dy, true, x, true, n, k, m, kF32, nullptr, nullptr, skpart, nullptr, 0.f, k, splits, st,
                              fused_db ? part : nullptr, 0)))
                return rc;
            const int64_t n4 = n * k / 4;
            splitk_reduce_kernel<<<unsigned(std::min<int64_t>((n4 + 31) / 32, 8 * kNumSMs)), 256, 0, st>>>(
                reinterpret_cast<const float4*>(skpart), n4, splits, reinterpret_cast<float4*>(dw));
            AFFMAE_LAUNCH_CHECK("splitk_reduce_kernel");
            if (fused_db) {
                colsum_final_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, st>>>(part, n, splits, db);
                AFFMAE_LAUNCH_CHECK("linear bwd bias");
            }
        }
    }
    if (db && !fused_db) {
        const int64_t rows_per = (m + kColsumChunks - 1) / kColsumChunks;
        const int64_t chunks = (m + rows_per - 1) / rows_per;
        const int groups = int(std::min<int64_t>(n / 8, kColsumThreads));
        const size_t shm = size_t(kColsumThreads / groups) * 8 * groups * sizeof(float);
        colsum_partial_kernel<<<unsigned(chunks), kColsumThreads, shm, st>>>(static_cast<const __nv_bfloat16*>(dy), m,
                                                                           n, rows_per, part);
        colsum_final_kernel<<<unsigned((n * 32 + 255) / 256), 256, 0, st>>>(part, n, int(chunks), db);
        AFFMAE_LAUNCH_CHECK("linear bwd bias");
    }
    return AFFMAE_OK;
}

int gelu_bwd(const void* pre, const void* dy, int64_t n, void* dpre, void* stream) {
    if (!pre || !dy || !dpre) return fail(AFFMAE_ECONFIG, "gelu_bwd: null pointer");
    if (n < 0 || n % 8) return fail(AFFMAE_EUNSUPPORTED, "gelu_bwd: element count must be a multiple of 8");
    if (n == 0) return AFFMAE_OK;
    const int64_t n8 = n / 8;
    const unsigned nb = unsigned(std::max<int64_t>(1, std::min<int64_t>((n8 + 255) / 256, 8 * kNumSMs)));
    gelu_bwd_kernel<<<nb, 256, 0, as_stream(stream)>>>(static_cast<const uint4*>(pre), static_cast<const uint4*>(dy),
                                                       n8, static_cast<uint4*>(dpre));
    AFFMAE_LAUNCH_CHECK("gelu_bwd_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
