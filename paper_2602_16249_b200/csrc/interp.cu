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
    float s = 0.f;  // normaliser in neighbour order (slots >= k hold 0: stop at k, k is uniform)
#pragma unroll
    for (int t = 0; t < kInterpMaxK; ++t) {
        if (t >= k) break;
        s += __shfl_sync(0xffffffffu, R.w[t / G::LPR], base + t % G::LPR);
    }
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
    // neighbour-outer: each neighbour's weight and id are shuffled once for all of the lane's
    // chunks (the chunk-outer order repeated both shuffles per chunk; the kernel is issue-bound)
    float acc[G::CPL][8];
#pragma unroll
    for (int cc = 0; cc < G::CPL; ++cc)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[cc][i] = 0.f;
#pragma unroll 8
    for (int t = 0; t < kInterpMaxK; ++t) {
        if (t >= k) break;  // uniform
        const float wt = __shfl_sync(0xffffffffu, R.w[t / G::LPR], base + t % G::LPR);
        const int jt = __shfl_sync(0xffffffffu, R.j[t / G::LPR], base + t % G::LPR);
        if (wt != 0.f) {
#pragma unroll
            for (int cc = 0; cc < G::CPL; ++cc) {
                float f[8];
                bf8_to_f32(__ldg(fb + int64_t(jt) * CPR + sl + cc * G::LPR), f);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[cc][i] = fmaf(wt, f[i], acc[cc][i]);
            }
        }
    }
    if (ok) {
#pragma unroll
        for (int cc = 0; cc < G::CPL; ++cc) out[rw * CPR + sl + cc * G::LPR] = f32_to_bf8(acc[cc]);
    }
}

template <int CPR, bool SCATTER>
__global__ void __launch_bounds__(256) interp_bwd_kernel(const float2* __restrict__ queries,
                                                         const float2* __restrict__ key_xy,
                                                         const uint4* __restrict__ feats,
                                                         const int32_t* __restrict__ idx,
                                                         const uint8_t* __restrict__ valid, int64_t batch,
                                                         int64_t nq, int64_t nk, int k, const float* __restrict__ p_ptr,
                                                         float eps, const uint4* __restrict__ dout,
                                                         float* __restrict__ dfeats, float* __restrict__ dp,
                                                         float2* __restrict__ dqueries, float* __restrict__ wout) {
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
                if (SCATTER) {
                    float* dst = dfb + int64_t(jt) * D + ch * 8;
                    red_add_v4(dst, wt * g[cc][0], wt * g[cc][1], wt * g[cc][2], wt * g[cc][3]);
                    red_add_v4(dst + 4, wt * g[cc][4], wt * g[cc][5], wt * g[cc][6], wt * g[cc][7]);
                }
            }
        }
#pragma unroll
        for (int o = G::LPR / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
#pragma unroll
        for (int i = 0; i < G::MPL; ++i)
            if (t == sl + i * G::LPR) dw[i] = part;
    }
    if (!SCATTER && ok) {  // the gather pass reads the weights back (0 for invalid slots)
#pragma unroll
        for (int i = 0; i < G::MPL; ++i)
            if (sl + i * G::LPR < k) wout[rw * k + sl + i * G::LPR] = R.w[i];
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
        interp_bwd_kernel<CPR_, true><<<interp_blocks<CPR_>(batch * nq), 256, 0, st>>>(                      \
            q2, k2, f, idx, valid, batch, nq, nk, int(k), p, float(eps), g, dfeats, dp, dq2, nullptr);       \
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

// ---------------------------------------------------------------------------
// Gather backward: dfeats from a reverse CSR of the knn rows (key -> the (row, slot)
// entries naming it) instead of scattered fp32 reductions.  The query pass writes
// the softmax weights; rev_count / rev_scan / rev_fill build the CSR per call (the
// rows change every call); interp_gather_kernel owns each key row (LPR lanes, CPL
// chunks each), sums w * g over its entries and adds the result once.
__global__ void interp_rev_count_kernel(const int32_t* __restrict__ idx, const uint8_t* __restrict__ valid,
                                        int64_t rows, int64_t nq, int64_t nk, int k, int32_t* __restrict__ cnt) {
    // entries < 2^31 (checked by the callers): 32-bit index math, the image from one division
    const uint32_t n = uint32_t(rows * k), span = uint32_t(nq * k);
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
        if (valid[e]) {
            // neighbouring rows share keys: one atomic per distinct key of the warp
            const int64_t slot = int64_t(e / span) * (nk + 1) + idx[e];
            const unsigned peers = __match_any_sync(__activemask(), (unsigned long long)slot);
            if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(cnt + slot, __popc(peers));
        }
}

// Per-image exclusive scan of the key counts, in place: one 1024-thread block per image walks
// its nk counts in coalesced tiles of 1024 (one per thread), carrying the running total;
// cnt[b*(nk+1) + j] -> offset of key j inside image b's entry range, cnt[b*(nk+1) + nk] = total.
__global__ void __launch_bounds__(1024) interp_rev_scan_kernel(int32_t* __restrict__ cnt, int64_t nk) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    int32_t* c = cnt + int64_t(blockIdx.x) * (nk + 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t t0 = 0; t0 < nk; t0 += 1024) {
        const int64_t i = t0 + threadIdx.x;
        const int32_t v = i < nk ? c[i] : 0;
        int32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            int32_t t = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            wsum[lane] = t;
        }
        __syncthreads();
        const int32_t base = carry;
        if (i < nk) c[i] = base + inc - v + (warp > 0 ? wsum[warp - 1] : 0);
        __syncthreads();
        if (threadIdx.x == 0) carry = base + wsum[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) c[nk] = carry;
}

__global__ void interp_rev_fill_kernel(const int32_t* __restrict__ idx, const uint8_t* __restrict__ valid,
                                       int64_t rows, int64_t nq, int64_t nk, int k, const int32_t* __restrict__ off,
                                       int32_t* __restrict__ cur, int32_t* __restrict__ ent,
                                       int32_t* __restrict__ ent_key) {
    const uint32_t n = uint32_t(rows * k), span = uint32_t(nq * k);
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
        if (valid[e]) {
            const int64_t b = e / span, j = idx[e];
            const unsigned peers = __match_any_sync(__activemask(), (unsigned long long)(b * nk + j));
            const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
            int32_t base = 0;
            if (lane == leader) base = atomicAdd(cur + b * nk + j, __popc(peers));
            base = __shfl_sync(peers, base, leader);
            const int64_t pos = b * nq * k + off[b * (nk + 1) + j] + base + __popc(peers & ((1u << lane) - 1u));
            ent[pos] = int32_t(e);
            ent_key[pos] = int32_t(b * nk + j);
        }
}

// Balanced gather: warps walk the key-sorted entry array in fixed chunks of 32 (lanes over
// the D dims, VPL each), so a key named by thousands of queries (the Perlin mask's border
// tokens) is spread over many warps.  A chunk loads its 32 entries, weights and keys with
// one instruction each, accumulates w * g while the key stays the same and flushes the
// running row with one vector reduction per lane at each key change (~2 flushes per chunk
// instead of one reduction per (entry, dim chunk) in the scattered backward).
template <int D>
__global__ void __launch_bounds__(256) interp_gather_kernel(const int32_t* __restrict__ off,
                                                            const int32_t* __restrict__ ent,
                                                            const int32_t* __restrict__ ent_key,
                                                            const float* __restrict__ w, int64_t batch, int64_t nq,
                                                            int64_t nk, int k, const __nv_bfloat16* __restrict__ dout,
                                                            float* __restrict__ dfeats) {
    constexpr int VPL = D / 32;
    static_assert(VPL % 2 == 0, "VPL");
    const int lane = threadIdx.x & 31;
    const int64_t span = nq * k, total = batch * span, nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
    auto flush = [&](int32_t key, float (&acc)[VPL]) {
        float* d = dfeats + int64_t(key) * D + lane * VPL;
        if constexpr (VPL % 4 == 0) {
#pragma unroll
            for (int c = 0; c < VPL; c += 4) red_add_v4(d + c, acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
        } else {
            atomicAdd(d, acc[0]);
            atomicAdd(d + 1, acc[1]);
        }
#pragma unroll
        for (int i = 0; i < VPL; ++i) acc[i] = 0.f;
    };
    for (int64_t c0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; c0 < total; c0 += nwarps * 32) {
        const int64_t pos = c0 + lane;
        int32_t mkey = -1, mrow = 0;
        float mw = 0.f;
        if (pos < total) {
            const int64_t b = pos / span;
            if (pos - b * span < off[b * (nk + 1) + nk]) {
                const int32_t e = __ldg(ent + pos);
                mkey = __ldg(ent_key + pos);
                mw = __ldg(w + e);
                mrow = e / k;
            }
        }
        if (__ballot_sync(0xffffffffu, mkey >= 0) == 0u) continue;
        float acc[VPL];
#pragma unroll
        for (int i = 0; i < VPL; ++i) acc[i] = 0.f;
        int32_t cur = -1;
#pragma unroll 4
        for (int u = 0; u < 32; ++u) {
            const int32_t key = __shfl_sync(0xffffffffu, mkey, u);
            const int32_t row = __shfl_sync(0xffffffffu, mrow, u);
            const float wt = __shfl_sync(0xffffffffu, mw, u);
            if (key < 0) continue;  // uniform
            if (key != cur) {
                if (cur >= 0) flush(cur, acc);
                cur = key;
            }
            const __nv_bfloat16* g = dout + int64_t(row) * D + lane * VPL;
#pragma unroll
            for (int c = 0; c < VPL; c += 2) {
                const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(g + c));
                acc[c] = fmaf(wt, t.x, acc[c]);
                acc[c + 1] = fmaf(wt, t.y, acc[c + 1]);
            }
        }
        if (cur >= 0) flush(cur, acc);
    }
}

// Reverse CSR of B images' neighbour rows idx/valid [B, nq, k] over nk keys, in caller
// buffers: off [B, nk+1] (per-image offsets), cur [B, nk] (scratch), ent / ent_key
// [B*nq*k] (image b's entries at b*nq*k + off, sorted by key; ent = global row*k + slot,
// ent_key = global key).  Shared with the decoder attention backward (gattn.cu).
void rev_csr_build(const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t nq, int64_t nk, int k,
                   int32_t* off, int32_t* cur, int32_t* ent, int32_t* ent_key, cudaStream_t st) {
    const int64_t ents = batch * nq * k;
    cudaMemsetAsync(off, 0, size_t(batch * (nk + 1)) * 4, st);
    cudaMemsetAsync(cur, 0, size_t(batch * nk) * 4, st);
    const unsigned eb = unsigned(std::max<int64_t>(1, std::min<int64_t>((ents + 255) / 256, 8 * kNumSMs)));
    interp_rev_count_kernel<<<eb, 256, 0, st>>>(idx, valid, batch * nq, nq, nk, k, off);
    interp_rev_scan_kernel<<<unsigned(batch), 1024, 0, st>>>(off, nk);
    interp_rev_fill_kernel<<<eb, 256, 0, st>>>(idx, valid, batch * nq, nq, nk, k, off, cur, ent, ent_key);
}

size_t interp_bwd_gather_workspace(int64_t batch, int64_t nq, int64_t nk, int64_t k) {
    const int64_t keys = batch * nk, ents = batch * nq * k;
    return size_t(batch * (nk + 1) + keys + 2 * ents) * 4 + size_t(ents) * 4 + 1024;
}

int interp_bwd_gather(const float* queries, const float* key_coords, const void* feats, const int32_t* idx,
                      const uint8_t* valid, int64_t batch, int64_t nq, int64_t nk, int64_t dim, int64_t k,
                      const float* p, double eps, const void* dout, float* dfeats, float* dp, float* dqueries,
                      void* workspace, size_t ws_bytes, void* stream) {
    int rc = interp_check(batch, nq, nk, dim, k);
    if (rc) return rc;
    if (!queries || !key_coords || !feats || !idx || !valid || !p || !dout || !dfeats || !dp || !dqueries)
        return fail(AFFMAE_ECONFIG, "interp bwd: null pointer");
    if (batch * nq * k >= (int64_t(1) << 31)) return fail(AFFMAE_EUNSUPPORTED, "interp bwd: more than 2^31 entries");
    if (!workspace || ws_bytes < interp_bwd_gather_workspace(batch, nq, nk, k))
        return fail(AFFMAE_ECONFIG, "interp bwd: workspace too small");
    if (batch * nq == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const int64_t keys = batch * nk, ents = batch * nq * k;
    int32_t* off = static_cast<int32_t*>(workspace);  // [B, nk + 1] per-image offsets
    int32_t* cur = off + batch * (nk + 1);
    int32_t* ent = cur + keys;
    int32_t* ent_key = ent + ents;
    float* wbuf = reinterpret_cast<float*>(ent_key + ents);
    rev_csr_build(idx, valid, batch, nq, nk, int(k), off, cur, ent, ent_key, st);
    const auto* q2 = reinterpret_cast<const float2*>(queries);
    const auto* k2 = reinterpret_cast<const float2*>(key_coords);
    const auto* f = static_cast<const uint4*>(feats);
    const auto* g = static_cast<const uint4*>(dout);
    auto* dq2 = reinterpret_cast<float2*>(dqueries);
#define AFFMAE_IG(CPR_)                                                                                      \
    case CPR_ * 8:                                                                                           \
        interp_bwd_kernel<CPR_, false><<<interp_blocks<CPR_>(batch * nq), 256, 0, st>>>(                     \
            q2, k2, f, idx, valid, batch, nq, nk, int(k), p, float(eps), g, dfeats, dp, dq2, wbuf);          \
        interp_gather_kernel<CPR_ * 8><<<unsigned(std::min<int64_t>((ents + 255) / 256, 16 * kNumSMs)), 256, 0, st>>>( \
            off, ent, ent_key, wbuf, batch, nq, nk, int(k), static_cast<const __nv_bfloat16*>(dout), dfeats); \
        break;
    switch (dim) {
        AFFMAE_IG(8)
        AFFMAE_IG(16)
        AFFMAE_IG(32)
        AFFMAE_IG(64)
    }
#undef AFFMAE_IG
    AFFMAE_LAUNCH_CHECK("interp_bwd_gather");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
