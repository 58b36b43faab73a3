// Softmax interpolation over fixed neighbour rows (make_interp_op,
// proj/include/affmae/interpolation.hpp:60; proj/src/interpolation.cpp:51-67,
// 93-142, 192-251) -- the decoder / deep-supervision upsampling of SURVEY.md
// §8(f) #2, batched over images on the B200.
//
// Forward, per query q with valid neighbours i (knn rows, idx/valid [B,Q,K]):
//   d_i = |q - x_i| + eps,  w = softmax(-p d),  out_q = sum_i w_i f_i.
// Backward (CustomOp semantics: += into the gradients):
//   df_i += w_i g,  dp += sum_i w_i (g.f_i - sum_j w_j g.f_j)(-d_i),
//   dq += sum_i (that)(-p)(q - x_i)/r_i  (zero subgradient at r_i = 0).
//
// Layout: a row of D bf16 is CPR = D/8 16-byte chunks; LPR = min(CPR, 16)
// lanes own one query row (CPL chunks each), RPW = 32/LPR rows per warp.
// Lane slot t (t = sl, sl + LPR, ...) computes neighbour t's distance and
// softmax weight; weights and indices reach the other lanes by shuffles, the
// normaliser is summed in neighbour order.  Neighbour rows are read with
// 16-byte loads, all of a row's members issued before use.  The backward
// scatters df with vector fp32 reductions (red.global.add.v4.f32): a key is
// the neighbour of several queries, so dfeats is fp32 and accumulation order
// is not fixed (deterministic to rounding, not bitwise).
#include <algorithm>

#include "common.cuh"

namespace affmae_b200 {

constexpr int kInterpMaxK = 32;

template <int CPR>
struct InterpGeo {
    static constexpr int LPR = CPR < 16 ? CPR : 16;
    static constexpr int RPW = 32 / LPR;
    static constexpr int CPL = CPR / LPR;
    static constexpr int MPL = (kInterpMaxK + LPR - 1) / LPR;  // neighbour slots per lane
};

__device__ __forceinline__ void bf8_to_f32(const uint4& v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
__device__ __forceinline__ uint4 f32_to_bf8(const float (&f)[8]) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

// Weights of one query row.  Lane slot t < k holds (neighbour id, weight,
// distance, r, dx, dy) of neighbour t; invalid slots have weight 0.  Returns
// the row's number of valid neighbours (0: the row gets no output / gradient).
template <int CPR>
struct InterpRow {
    static constexpr int MPL = InterpGeo<CPR>::MPL;
    int j[MPL];
    float w[MPL], d[MPL], r[MPL], dx[MPL], dy[MPL];
    int nvalid;
};

template <int CPR>
__device__ __forceinline__ void interp_row_weights(InterpRow<CPR>& R, const float2* kxy, const int32_t* idx,
                                                   const uint8_t* valid, int k, float2 q, float p, float eps,
                                                   bool ok, int lane) {
    using G = InterpGeo<CPR>;
    const int sl = lane % G::LPR, base = lane - sl;
    float mx = -INFINITY;
    int nv = 0;
#pragma unroll
    for (int i = 0; i < G::MPL; ++i) {
        const int t = sl + i * G::LPR;
        const bool v = ok && t < k && valid[t] != 0;
        R.j[i] = v ? idx[t] : 0;
        const float2 x = v ? __ldg(kxy + R.j[i]) : q;
        R.dx[i] = q.x - x.x;
        R.dy[i] = q.y - x.y;
        R.r[i] = sqrtf(fmaf(R.dx[i], R.dx[i], R.dy[i] * R.dy[i]));
        R.d[i] = R.r[i] + eps;
        R.w[i] = v ? -p * R.d[i] : -INFINITY;  // logit
        mx = fmaxf(mx, R.w[i]);
        nv += v;
    }
#pragma unroll
    for (int o = G::LPR / 2; o > 0; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        nv += __shfl_xor_sync(0xffffffffu, nv, o);
    }
#pragma unroll
    for (int i = 0; i < G::MPL; ++i) R.w[i] = R.w[i] == -INFINITY ? 0.f : __expf(R.w[i] - mx);
    float s = 0.f;  // normaliser in neighbour order
#pragma unroll
    for (int t = 0; t < kInterpMaxK; ++t) s += __shfl_sync(0xffffffffu, R.w[t / G::LPR], base + t % G::LPR);
    const float is = nv > 0 ? 1.f / s : 0.f;
#pragma unroll
    for (int i = 0; i < G::MPL; ++i) R.w[i] *= is;
    R.nvalid = nv;
}

template <int CPR>
__global__ void __launch_bounds__(256) interp_fwd_kernel(const float2* __restrict__ queries,
                                                         const float2* __restrict__ key_xy,
                                                         const uint4* __restrict__ feats,
                                                         const int32_t* __restrict__ idx,
                                                         const uint8_t* __restrict__ valid, int64_t batch,
                                                         int64_t nq, int64_t nk, int k, const float* __restrict__ p_ptr,
                                                         float eps, uint4* __restrict__ out) {
    using G = InterpGeo<CPR>;
    const int lane = threadIdx.x & 31, sl = lane % G::LPR, base = lane - sl;
    const int64_t row = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * G::RPW + lane / G::LPR;
    const bool ok = row < batch * nq;
    const int64_t rw = ok ? row : 0, b = rw / nq;
    const float p = *p_ptr;
    InterpRow<CPR> R;
    interp_row_weights<CPR>(R, key_xy + b * nk, idx + rw * k, valid + rw * k, k, queries[rw], p, eps, ok, lane);
    const uint4* fb = feats + b * nk * CPR;
#pragma unroll
    for (int cc = 0; cc < G::CPL; ++cc) {
        const int ch = sl + cc * G::LPR;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
        for (int t = 0; t < kInterpMaxK; ++t) {
            if (t >= k) break;  // uniform
            const float wt = __shfl_sync(0xffffffffu, R.w[t / G::LPR], base + t % G::LPR);
            const int jt = __shfl_sync(0xffffffffu, R.j[t / G::LPR], base + t % G::LPR);
            if (wt != 0.f) {
                float f[8];
                bf8_to_f32(__ldg(fb + int64_t(jt) * CPR + ch), f);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = fmaf(wt, f[i], acc[i]);
            }
        }
        if (ok) out[rw * CPR + ch] = f32_to_bf8(acc);
    }
}

template <int CPR>
__global__ void __launch_bounds__(256) interp_bwd_kernel(const float2* __restrict__ queries,
                                                         const float2* __restrict__ key_xy,
                                                         const uint4* __restrict__ feats,
                                                         const int32_t* __restrict__ idx,
                                                         const uint8_t* __restrict__ valid, int64_t batch,
                                                         int64_t nq, int64_t nk, int k, const float* __restrict__ p_ptr,
                                                         float eps, const uint4* __restrict__ dout,
                                                         float* __restrict__ dfeats, float* __restrict__ dp,
                                                         float2* __restrict__ dqueries) {
    using G = InterpGeo<CPR>;
    constexpr int D = CPR * 8;
    const int lane = threadIdx.x & 31, sl = lane % G::LPR, base = lane - sl;
    const int64_t row = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * G::RPW + lane / G::LPR;
    const bool ok = row < batch * nq;
    const int64_t rw = ok ? row : 0, b = rw / nq;
    const float p = *p_ptr;
    InterpRow<CPR> R;
    interp_row_weights<CPR>(R, key_xy + b * nk, idx + rw * k, valid + rw * k, k, queries[rw], p, eps, ok, lane);
    const uint4* fb = feats + b * nk * CPR;
    float* dfb = dfeats + b * nk * D;
    float g[G::CPL][8];
#pragma unroll
    for (int cc = 0; cc < G::CPL; ++cc) bf8_to_f32(ok ? __ldg(dout + rw * CPR + sl + cc * G::LPR) : make_uint4(0, 0, 0, 0), g[cc]);
    // dw_t = <g, f_t> for the lane's neighbour slots; df_t = w_t g scattered
    float dw[G::MPL];
#pragma unroll
    for (int i = 0; i < G::MPL; ++i) dw[i] = 0.f;
#pragma unroll 4
    for (int t = 0; t < kInterpMaxK; ++t) {
        if (t >= k) break;  // uniform
        const float wt = __shfl_sync(0xffffffffu, R.w[t / G::LPR], base + t % G::LPR);
        const int jt = __shfl_sync(0xffffffffu, R.j[t / G::LPR], base + t % G::LPR);
        float part = 0.f;
        if (wt != 0.f) {
#pragma unroll
            for (int cc = 0; cc < G::CPL; ++cc) {
                const int ch = sl + cc * G::LPR;
                float f[8];
                bf8_to_f32(__ldg(fb + int64_t(jt) * CPR + ch), f);
#pragma unroll
                for (int i = 0; i < 8; ++i) part = fmaf(g[cc][i], f[i], part);
                float* dst = dfb + int64_t(jt) * D + ch * 8;
                red_add_v4(dst, wt * g[cc][0], wt * g[cc][1], wt * g[cc][2], wt * g[cc][3]);
                red_add_v4(dst + 4, wt * g[cc][4], wt * g[cc][5], wt * g[cc][6], wt * g[cc][7]);
            }
        }
#pragma unroll
        for (int o = G::LPR / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
#pragma unroll
        for (int i = 0; i < G::MPL; ++i)
            if (t == sl + i * G::LPR) dw[i] = part;
    }
    float wdot = 0.f;
#pragma unroll
    for (int i = 0; i < G::MPL; ++i) wdot = fmaf(R.w[i], dw[i], wdot);
#pragma unroll
    for (int o = G::LPR / 2; o > 0; o >>= 1) wdot += __shfl_xor_sync(0xffffffffu, wdot, o);
    float lp = 0.f, qx = 0.f, qy = 0.f;
#pragma unroll
    for (int i = 0; i < G::MPL; ++i) {
        const float dl = R.w[i] * (dw[i] - wdot);
        lp = fmaf(dl, -R.d[i], lp);
        if (R.w[i] != 0.f && R.r[i] > 0.f) {
            const float dd = dl * -p / R.r[i];
            qx = fmaf(dd, R.dx[i], qx);
            qy = fmaf(dd, R.dy[i], qy);
        }
    }
#pragma unroll
    for (int o = G::LPR / 2; o > 0; o >>= 1) {
        lp += __shfl_xor_sync(0xffffffffu, lp, o);
        qx += __shfl_xor_sync(0xffffffffu, qx, o);
        qy += __shfl_xor_sync(0xffffffffu, qy, o);
    }
    if (ok && sl == 0 && R.nvalid > 0) {
        float2 cur = dqueries[rw];
        dqueries[rw] = make_float2(cur.x + qx, cur.y + qy);
    }
    // dp: rows -> warp -> block -> one atomic per block
    __shared__ float red[8];
    float v = (ok && sl == 0) ? lp : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
        atomicAdd(dp, s);
    }
}

static int interp_check(int64_t batch, int64_t nq, int64_t nk, int64_t dim, int64_t k) {
    if (batch < 0 || nq < 0 || nk < 1) return fail(AFFMAE_ECONFIG, "interp: bad sizes");
    if (k < 1 || k > kInterpMaxK) return fail(AFFMAE_EUNSUPPORTED, "interp: k must be in [1, 32]");
    if (dim != 64 && dim != 128 && dim != 256 && dim != 512)
        return fail(AFFMAE_EUNSUPPORTED, "interp: dim must be 64, 128, 256 or 512");
    return AFFMAE_OK;
}

template <int CPR>
static unsigned interp_blocks(int64_t rows) {
    constexpr int RPW = InterpGeo<CPR>::RPW;
    return unsigned(((rows + RPW - 1) / RPW + 7) / 8);
}

int interp_fwd(const float* queries, const float* key_coords, const void* feats, const int32_t* idx,
               const uint8_t* valid, int64_t batch, int64_t nq, int64_t nk, int64_t dim, int64_t k,
               const float* p, double eps, void* out, void* stream) {
    int rc = interp_check(batch, nq, nk, dim, k);
    if (rc) return rc;
    if (!queries || !key_coords || !feats || !idx || !valid || !p || !out)
        return fail(AFFMAE_ECONFIG, "interp: null pointer");
    if (batch * nq == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const auto* q2 = reinterpret_cast<const float2*>(queries);
    const auto* k2 = reinterpret_cast<const float2*>(key_coords);
    const auto* f = static_cast<const uint4*>(feats);
    auto* o = static_cast<uint4*>(out);
#define AFFMAE_IF(CPR_)                                                                                   \
    case CPR_ * 8:                                                                                        \
        interp_fwd_kernel<CPR_><<<interp_blocks<CPR_>(batch * nq), 256, 0, st>>>(q2, k2, f, idx, valid,   \
                                                                                 batch, nq, nk, int(k), p, \
                                                                                 float(eps), o);          \
        break;
    switch (dim) {
        AFFMAE_IF(8)
        AFFMAE_IF(16)
        AFFMAE_IF(32)
        AFFMAE_IF(64)
    }
#undef AFFMAE_IF
    AFFMAE_LAUNCH_CHECK("interp_fwd_kernel");
    return AFFMAE_OK;
}

int interp_bwd(const float* queries, const float* key_coords, const void* feats, const int32_t* idx,
               const uint8_t* valid, int64_t batch, int64_t nq, int64_t nk, int64_t dim, int64_t k,
               const float* p, double eps, const void* dout, float* dfeats, float* dp, float* dqueries,
               void* stream) {
    int rc = interp_check(batch, nq, nk, dim, k);
    if (rc) return rc;
    if (!queries || !key_coords || !feats || !idx || !valid || !p || !dout || !dfeats || !dp || !dqueries)
        return fail(AFFMAE_ECONFIG, "interp bwd: null pointer");
    if (batch * nq == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const auto* q2 = reinterpret_cast<const float2*>(queries);
    const auto* k2 = reinterpret_cast<const float2*>(key_coords);
    const auto* f = static_cast<const uint4*>(feats);
    const auto* g = static_cast<const uint4*>(dout);
    auto* dq2 = reinterpret_cast<float2*>(dqueries);
#define AFFMAE_IB(CPR_)                                                                                      \
    case CPR_ * 8:                                                                                           \
        interp_bwd_kernel<CPR_><<<interp_blocks<CPR_>(batch * nq), 256, 0, st>>>(                            \
            q2, k2, f, idx, valid, batch, nq, nk, int(k), p, float(eps), g, dfeats, dp, dq2);                \
        break;
    switch (dim) {
        AFFMAE_IB(8)
        AFFMAE_IB(16)
        AFFMAE_IB(32)
        AFFMAE_IB(64)
    }
#undef AFFMAE_IB
    AFFMAE_LAUNCH_CHECK("interp_bwd_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
