// Attention over arbitrary per-token neighbour rows: nbhd_attn_streaming /
// nbhd_attn_backward (include/affmae/attention.hpp:52-72; src/attention.cpp:
// 119-358) on a general NeighborIndex -- the decoder's cross attention over
// one_to_one rows and self attention over knn rows (src/pipeline.cpp:64-71,
// 495-535).  The encoder's cluster attention (attention.cu)
// exploits the shared key lists of a cluster; here every query has its own
// (short, width <= 31) list, so the layout is one warp per (query, head):
//   * scores: lane j holds key slot j (full head_dim dot product from its key
//     row, the query row broadcast), BiasNet evaluated exactly (tanh MLP of the
//     offset / patch), lane `width` holds the blank slot; softmax across lanes;
//   * values: lanes over head dims, neighbour weights and ids by shuffle;
//   * backward: dP and dS per lane slot, dq over dims, dk / dv scattered with
//     fp32 reductions (a key serves several queries), blank and BiasNet
//     parameter gradients reduced per warp, per block, then one atomic each.
#include "common.cuh"

namespace affmae_b200 {

constexpr int kGMaxHidden = 32;

struct GAttnP {
    const __nv_bfloat16 *q, *k, *v, *bk, *bv;
    const float* coords;
    const float *w1, *b1, *w2, *b2, *blank;
    const int32_t* idx;
    const uint8_t* valid;
    int64_t batch, n;
    int m, heads, hidden;
    float scale, inv_patch;
};

template <int HD>
struct GRow {  // a head_dim row, lanes over dims (HD / 32 values per lane; HD 16: lanes 0-15)
    static constexpr int PL = HD >= 32 ? HD / 32 : 1;
    static __device__ __forceinline__ bool on(int lane) { return HD >= 32 || lane < HD; }
};

__device__ __forceinline__ float gdot_row(const __nv_bfloat16* a, const __nv_bfloat16* b, int hd) {
    // full dot product of two hd-element bf16 rows by one thread (16-byte loads)
    float s = 0.f;
    for (int c = 0; c < hd; c += 8) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + c)), y = __ldg(reinterpret_cast<const uint4*>(b + c));
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&x);
        const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 u = __bfloat1622float2(xh[i]), w = __bfloat1622float2(yh[i]);
            s = fmaf(u.x, w.x, fmaf(u.y, w.y, s));
        }
    }
    return s;
}

__device__ __forceinline__ float gbias(const GAttnP& p, int h, float ox, float oy) {
    float acc = p.b2[h];
    for (int u = 0; u < p.hidden; ++u) {
        const float pre = fmaf(p.w1[h * 2 * p.hidden + u], ox, fmaf(p.w1[h * 2 * p.hidden + p.hidden + u], oy,
                                                                     p.b1[h * p.hidden + u]));
        acc = fmaf(p.w2[h * p.hidden + u], tanhf(pre), acc);
    }
    return acc;
}

// scores of the lane's slot (key slot lane < m, blank at lane m), softmax weight, key id
struct GSlot {
    float w;   // softmax weight (0 for invalid / unused lanes)
    int t;     // key token (image-local), -1 if none
    float ox, oy, s;
};

template <int HD>
__device__ __forceinline__ GSlot gattn_slot(const GAttnP& p, int64_t b, int64_t i, int h, int lane) {
    const int64_t ld = int64_t(p.heads) * HD;
    const __nv_bfloat16* qrow = p.q + (b * p.n + i) * ld + h * HD;
    const float2* xy = reinterpret_cast<const float2*>(p.coords) + b * p.n;
    GSlot sl{0.f, -1, 0.f, 0.f, -INFINITY};
    if (lane < p.m) {
        const int64_t e = (b * p.n + i) * p.m + lane;
        if (p.valid[e]) {
            sl.t = p.idx[e];
            const float2 qx = xy[i], kx = xy[sl.t];
            sl.ox = (kx.x - qx.x) * p.inv_patch;
            sl.oy = (kx.y - qx.y) * p.inv_patch;
            sl.s = p.scale * gdot_row(qrow, p.k + (b * p.n + sl.t) * ld + h * HD, HD) + gbias(p, h, sl.ox, sl.oy);
        }
    } else if (lane == p.m) {
        sl.s = p.scale * gdot_row(qrow, p.bk + h * HD, HD) + p.blank[h];
    }
    float mx = sl.s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float e = sl.s == -INFINITY ? 0.f : __expf(sl.s - mx);
    float l = e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    sl.w = e / l;
    sl.s = mx + __logf(l);  // lse (every lane)
    return sl;
}

template <int HD>
__global__ void __launch_bounds__(256) gattn_fwd_kernel(GAttnP p, __nv_bfloat16* __restrict__ out,
                                                        float* __restrict__ lse) {
    constexpr int PL = GRow<HD>::PL;
    const int lane = threadIdx.x & 31;
    const int64_t total = p.batch * p.n * p.heads, ws = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t ld = int64_t(p.heads) * HD;
    for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < total; w += ws) {
        const int h = int(w % p.heads);
        const int64_t bi = w / p.heads, b = bi / p.n, i = bi - b * p.n;
        const GSlot sl = gattn_slot<HD>(p, b, i, h, lane);
        float acc[PL];
#pragma unroll
        for (int r = 0; r < PL; ++r) acc[r] = 0.f;
        for (int j = 0; j < p.m; ++j) {
            const float wj = __shfl_sync(0xffffffffu, sl.w, j);
            const int tj = __shfl_sync(0xffffffffu, sl.t, j);
            if (tj >= 0) {
                const __nv_bfloat16* vr = p.v + (b * p.n + tj) * ld + h * HD;
#pragma unroll
                for (int r = 0; r < PL; ++r)
                    if (GRow<HD>::on(lane)) acc[r] = fmaf(wj, __bfloat162float(vr[lane + 32 * r]), acc[r]);
            }
        }
        const float wb = __shfl_sync(0xffffffffu, sl.w, p.m);
#pragma unroll
        for (int r = 0; r < PL && GRow<HD>::on(lane); ++r) {
            acc[r] = fmaf(wb, __bfloat162float(p.bv[h * HD + lane + 32 * r]), acc[r]);
            out[(b * p.n + i) * ld + h * HD + lane + 32 * r] = __float2bfloat16(acc[r]);
        }
        if (lane == 0) lse[bi * p.heads + h] = sl.s;
    }
}

template <int HD>
__global__ void __launch_bounds__(256) gattn_bwd_kernel(GAttnP p, const __nv_bfloat16* __restrict__ dout,
                                                        __nv_bfloat16* __restrict__ dq, float* __restrict__ dk,
                                                        float* __restrict__ dv, float* __restrict__ dbk,
                                                        float* __restrict__ dbv, float* __restrict__ dw1,
                                                        float* __restrict__ db1, float* __restrict__ dw2,
                                                        float* __restrict__ db2, float* __restrict__ dblank) {
    constexpr int PL = GRow<HD>::PL;
    __shared__ float pacc[8][4 * kGMaxHidden + 2];  // per warp: BiasNet grads of its head, blank param
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = 4 * p.hidden + 2;
    for (int e = lane; e < G; e += 32) pacc[warp][e] = 0.f;
    const int64_t total = p.batch * p.n * p.heads, ws = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t ld = int64_t(p.heads) * HD;
    // heads are the fastest index of the warp id and the grid is a multiple of heads
    // warps, so every warp of this block sees one fixed head (pacc is per head)
    int head_of_warp = -1;
    float bkacc[PL], bvacc[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) bkacc[r] = bvacc[r] = 0.f;
    for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < total; w += ws) {
        const int h = int(w % p.heads);
        head_of_warp = h;
        const int64_t bi = w / p.heads, b = bi / p.n, i = bi - b * p.n;
        const GSlot sl = gattn_slot<HD>(p, b, i, h, lane);
        const __nv_bfloat16* grow = dout + (b * p.n + i) * ld + h * HD;
        const __nv_bfloat16* qrow = p.q + (b * p.n + i) * ld + h * HD;
        // dP for the lane's slot
        float dP = 0.f;
        if (sl.t >= 0) dP = gdot_row(grow, p.v + (b * p.n + sl.t) * ld + h * HD, HD);
        else if (lane == p.m) dP = gdot_row(grow, p.bv + h * HD, HD);
        float D = sl.w * dP;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) D += __shfl_xor_sync(0xffffffffu, D, o);
        const float dS = sl.w * (dP - D);  // 0 on unused lanes
        // dq over dims, dk / dv scatter
        float qv[PL], gv[PL], dqa[PL];
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            const bool on = GRow<HD>::on(lane);
            qv[r] = on ? __bfloat162float(qrow[lane + 32 * r]) : 0.f;
            gv[r] = on ? __bfloat162float(grow[lane + 32 * r]) : 0.f;
            dqa[r] = 0.f;
        }
        for (int j = 0; j < p.m; ++j) {
            const float dSj = __shfl_sync(0xffffffffu, dS, j), wj = __shfl_sync(0xffffffffu, sl.w, j);
            const int tj = __shfl_sync(0xffffffffu, sl.t, j);
            if (tj < 0) continue;
            const __nv_bfloat16* kr = p.k + (b * p.n + tj) * ld + h * HD;
            float* dkr = dk + (b * p.n + tj) * ld + h * HD;
            float* dvr = dv + (b * p.n + tj) * ld + h * HD;
#pragma unroll
            for (int r = 0; r < PL && GRow<HD>::on(lane); ++r) {
                dqa[r] = fmaf(dSj, __bfloat162float(kr[lane + 32 * r]), dqa[r]);
                atomicAdd(dkr + lane + 32 * r, p.scale * dSj * qv[r]);
                atomicAdd(dvr + lane + 32 * r, wj * gv[r]);
            }
        }
        const float dSb = __shfl_sync(0xffffffffu, dS, p.m), wb = __shfl_sync(0xffffffffu, sl.w, p.m);
#pragma unroll
        for (int r = 0; r < PL && GRow<HD>::on(lane); ++r) {
            dqa[r] = fmaf(dSb, __bfloat162float(p.bk[h * HD + lane + 32 * r]), dqa[r]);
            dq[(b * p.n + i) * ld + h * HD + lane + 32 * r] = __float2bfloat16(p.scale * dqa[r]);
            bkacc[r] = fmaf(p.scale * dSb, qv[r], bkacc[r]);
            bvacc[r] = fmaf(wb, gv[r], bvacc[r]);
        }
        // BiasNet gradients of the pairs (lane = slot), reduced over the warp
        const bool pair = sl.t >= 0;
        for (int u = 0; u < p.hidden; ++u) {
            float gx = 0.f, gy = 0.f, gb = 0.f, gw = 0.f;
            if (pair) {
                const float pre = fmaf(p.w1[h * 2 * p.hidden + u], sl.ox,
                                       fmaf(p.w1[h * 2 * p.hidden + p.hidden + u], sl.oy, p.b1[h * p.hidden + u]));
                const float th = tanhf(pre);
                const float dpre = dS * p.w2[h * p.hidden + u] * (1.f - th * th);
                gx = dpre * sl.ox;
                gy = dpre * sl.oy;
                gb = dpre;
                gw = dS * th;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                gx += __shfl_xor_sync(0xffffffffu, gx, o);
                gy += __shfl_xor_sync(0xffffffffu, gy, o);
                gb += __shfl_xor_sync(0xffffffffu, gb, o);
                gw += __shfl_xor_sync(0xffffffffu, gw, o);
            }
            if (lane == 0) {
                pacc[warp][u] += gx;
                pacc[warp][p.hidden + u] += gy;
                pacc[warp][2 * p.hidden + u] += gb;
                pacc[warp][3 * p.hidden + u] += gw;
            }
        }
        float g2 = pair ? dS : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) g2 += __shfl_xor_sync(0xffffffffu, g2, o);
        if (lane == 0) {
            pacc[warp][4 * p.hidden] += g2;
            pacc[warp][4 * p.hidden + 1] += dSb;
        }
    }
    __syncwarp();
    if (head_of_warp >= 0) {
        const int h = head_of_warp;
#pragma unroll
        for (int r = 0; r < PL && GRow<HD>::on(lane); ++r) {
            atomicAdd(dbk + h * HD + lane + 32 * r, bkacc[r]);
            atomicAdd(dbv + h * HD + lane + 32 * r, bvacc[r]);
        }
        for (int e = lane; e < G; e += 32) {
            const float val = pacc[warp][e];
            const int H = p.hidden;
            if (e < H) atomicAdd(dw1 + h * 2 * H + e, val);
            else if (e < 2 * H) atomicAdd(dw1 + h * 2 * H + H + (e - H), val);
            else if (e < 3 * H) atomicAdd(db1 + h * H + (e - 2 * H), val);
            else if (e < 4 * H) atomicAdd(dw2 + h * H + (e - 3 * H), val);
            else if (e == 4 * H) atomicAdd(db2 + h, val);
            else atomicAdd(dblank + h, val);
        }
    }
}

static int gattn_fill(GAttnP& p, const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx,
                      const uint8_t* valid, int64_t batch, int64_t tokens, int64_t width) {
    if (!a || !in || !idx || !valid || !in->q || !in->k || !in->v || !in->blank_k || !in->blank_v || !in->coords ||
        !in->w1 || !in->b1 || !in->w2 || !in->b2 || !in->blank)
        return fail(AFFMAE_ECONFIG, "gattn: null pointer");
    if (a->head_dim != 16 && a->head_dim != 32 && a->head_dim != 64)
        return fail(AFFMAE_EUNSUPPORTED, "gattn: head_dim must be 16, 32 or 64");
    if (width < 1 || width > 31) return fail(AFFMAE_EUNSUPPORTED, "gattn: neighbourhood width must be in [1, 31]");
    if (a->bias_hidden < 1 || a->bias_hidden > kGMaxHidden) return fail(AFFMAE_EUNSUPPORTED, "gattn: bias_hidden");
    if (a->heads < 1 || !(a->patch > 0.0) || batch < 0 || tokens < 1) return fail(AFFMAE_ECONFIG, "gattn: bad shape");
    p.q = reinterpret_cast<const __nv_bfloat16*>(in->q);
    p.k = reinterpret_cast<const __nv_bfloat16*>(in->k);
    p.v = reinterpret_cast<const __nv_bfloat16*>(in->v);
    p.bk = reinterpret_cast<const __nv_bfloat16*>(in->blank_k);
    p.bv = reinterpret_cast<const __nv_bfloat16*>(in->blank_v);
    p.coords = in->coords;
    p.w1 = in->w1;
    p.b1 = in->b1;
    p.w2 = in->w2;
    p.b2 = in->b2;
    p.blank = in->blank;
    p.idx = idx;
    p.valid = valid;
    p.batch = batch;
    p.n = tokens;
    p.m = int(width);
    p.heads = a->heads;
    p.hidden = a->bias_hidden;
    p.scale = float(1.0 / std::sqrt(double(a->head_dim)));
    p.inv_patch = float(1.0 / a->patch);
    return AFFMAE_OK;
}

static unsigned gattn_blocks(int64_t warps, int heads) {
    // 8 warps per block; a whole number of head cycles per grid stride (heads | 8*blocks)
    int64_t nb = std::min<int64_t>((warps + 7) / 8, 8 * kNumSMs);
    nb = std::max<int64_t>(nb, 1);
    while ((nb * 8) % heads) ++nb;
    return unsigned(nb);
}

int gattn_fwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx, const uint8_t* valid,
              int64_t batch, int64_t tokens, int64_t width, void* out, float* lse, void* stream) {
    GAttnP p{};
    int rc = gattn_fill(p, a, in, idx, valid, batch, tokens, width);
    if (rc) return rc;
    if (!out || !lse) return fail(AFFMAE_ECONFIG, "gattn: null output");
    if (batch == 0) return AFFMAE_OK;
    const unsigned nb = gattn_blocks(batch * tokens * a->heads, a->heads);
    auto* o = static_cast<__nv_bfloat16*>(out);
    if (a->head_dim == 16) gattn_fwd_kernel<16><<<nb, 256, 0, as_stream(stream)>>>(p, o, lse);
    else if (a->head_dim == 32) gattn_fwd_kernel<32><<<nb, 256, 0, as_stream(stream)>>>(p, o, lse);
    else gattn_fwd_kernel<64><<<nb, 256, 0, as_stream(stream)>>>(p, o, lse);
    AFFMAE_LAUNCH_CHECK("gattn_fwd_kernel");
    return AFFMAE_OK;
}

int gattn_bwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx, const uint8_t* valid,
              int64_t batch, int64_t tokens, int64_t width, const void* dout, void* dq, float* dk, float* dv,
              float* dbk, float* dbv, float* dw1, float* db1, float* dw2, float* db2, float* dblank, void* stream) {
    GAttnP p{};
    int rc = gattn_fill(p, a, in, idx, valid, batch, tokens, width);
    if (rc) return rc;
    if (!dout || !dq || !dk || !dv || !dbk || !dbv || !dw1 || !db1 || !dw2 || !db2 || !dblank)
        return fail(AFFMAE_ECONFIG, "gattn bwd: null output");
    if (batch == 0) return AFFMAE_OK;
    const unsigned nb = gattn_blocks(batch * tokens * a->heads, a->heads);
    const auto* g = static_cast<const __nv_bfloat16*>(dout);
    auto* q = static_cast<__nv_bfloat16*>(dq);
    if (a->head_dim == 16)
        gattn_bwd_kernel<16><<<nb, 256, 0, as_stream(stream)>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    else if (a->head_dim == 32)
        gattn_bwd_kernel<32><<<nb, 256, 0, as_stream(stream)>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    else
        gattn_bwd_kernel<64><<<nb, 256, 0, as_stream(stream)>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    AFFMAE_LAUNCH_CHECK("gattn_bwd_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
