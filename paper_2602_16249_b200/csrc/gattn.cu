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
constexpr int kGMaxHeads = 8;  // a block is heads warps (<= 256 threads)

struct GAttnP {
    const __nv_bfloat16 *q, *k, *v, *bk, *bv;
    const float* coords;
    const float *w1, *b1, *w2, *b2, *blank;
    const int32_t* idx;
    const uint8_t* valid;
    int64_t batch, n;
    int m, heads, hidden;
    float scale, inv_patch;
    float2* dsw;  // backward gather mode: {scale dS, w} per (entry, head); nullptr = scatter dk / dv
    int o2o;      // backward: row i's only key is token i (bf16 dk / dv stored directly)
    // row strides (elements): q rows, k / v rows, and the bf16 gradient outputs dq (and the
    // one-to-one dk / dv): D for dense tensors, 3D / 2D when they are column slices of one
    // fused QKV / KV projection.  out / dout / fp32 dk, dv are always dense.
    int64_t ldq, ldkv, ldd, lddkv;
    float* part;  // row backward: per-block parameter-gradient rows (fixed-order reduce), else atomics
    int part_blocks;  // rows in `part` (caps the grid)
};

// destination of element e of a row-backward parameter-gradient row
// [D] dbk | [D] dbv | [H][hid][4] BiasNet {w1x, w1y, b1, w2} | [H] db2 | [H] dblank
__device__ __forceinline__ float* grad_dst(int e, int D, int H, int hid, float* dbk, float* dbv, float* dw1,
                                           float* db1, float* dw2, float* db2, float* dblank) {
    if (e < D) return dbk + e;
    if (e < 2 * D) return dbv + (e - D);
    if (e < 2 * D + 4 * H * hid) {
        const int r = e - 2 * D, hu = r >> 2, c = r & 3, hh = hu / hid, u = hu - hh * hid;
        return c == 0 ? dw1 + hh * 2 * hid + u : c == 1 ? dw1 + hh * 2 * hid + hid + u
             : c == 2 ? db1 + hh * hid + u : dw2 + hh * hid + u;
    }
    if (e < 2 * D + 4 * H * hid + H) return db2 + (e - 2 * D - 4 * H * hid);
    return dblank + (e - 2 * D - 4 * H * hid - H);
}
// sum of the per-block rows in block order, added once per element (deterministic)
__global__ void grow_reduce_kernel(const float* __restrict__ part, int blocks, int W, int D, int H, int hid,
                                   float* dbk, float* dbv, float* dw1, float* db1, float* dw2, float* db2,
                                   float* dblank) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= W) return;
    float v = 0.f;
    for (int b = 0; b < blocks; ++b) v += part[size_t(b) * W + e];
    *grad_dst(e, D, H, hid, dbk, dbv, dw1, db1, dw2, db2, dblank) += v;
}

__device__ __forceinline__ void gred_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

template <int HD>
__device__ __forceinline__ void gload_row(const __nv_bfloat16* r, float (&f)[HD], float mul) {
#pragma unroll
    for (int c = 0; c < HD; c += 8) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(r + c));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 t = __bfloat1622float2(h[i]);
            f[c + 2 * i] = t.x * mul;
            f[c + 2 * i + 1] = t.y * mul;
        }
    }
}

template <int HD>
__device__ __forceinline__ float gdot(const float (&a)[HD], const __nv_bfloat16* r) {
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < HD; c += 8) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(r + c));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 t = __bfloat1622float2(h[i]);
            s = fmaf(a[c + 2 * i], t.x, fmaf(a[c + 2 * i + 1], t.y, s));
        }
    }
    return s;
}

// BiasNet of one pair from the head's units {w1x, w1y, b1, w2} in shared memory
__device__ __forceinline__ float gbias(const float4* un, int hidden, float b2, float ox, float oy) {
    float acc = b2;
    for (int u = 0; u < hidden; ++u) {
        const float4 w = un[u];
        acc = fmaf(w.w, tanh_fast(fmaf(w.x, ox, fmaf(w.y, oy, w.z))), acc);
    }
    return acc;
}

__device__ __forceinline__ void gstage_units(const GAttnP& p, float4* units) {
    const int H = p.hidden;
    for (int e = threadIdx.x; e < p.heads * H; e += blockDim.x) {
        const int h = e / H, u = e - h * H;
        units[e] = make_float4(p.w1[h * 2 * H + u], p.w1[h * 2 * H + H + u], p.b1[h * H + u], p.w2[h * H + u]);
    }
    __syncthreads();
}

// Thread per (token, head): a block is heads warps over a tile of 32 tokens, warp = head,
// lane = token, so a warp's BiasNet / blank gradients belong to one head and the heads'
// 2*HD-byte row segments of one key are read by the same block.
template <int HD>
__global__ void __launch_bounds__(256) gattn_fwd_kernel(GAttnP p, __nv_bfloat16* __restrict__ out,
                                                         float* __restrict__ lse) {
    extern __shared__ float4 g_units[];
    gstage_units(p, g_units);
    const int lane = threadIdx.x & 31, h = threadIdx.x >> 5;
    const float4* un = g_units + h * p.hidden;
    const float b2 = p.b2[h], blank = p.blank[h];
    const int64_t ntok = p.batch * p.n, ld = int64_t(p.heads) * HD;
    const float2* xy = reinterpret_cast<const float2*>(p.coords);
    for (int64_t gi = int64_t(blockIdx.x) * 32 + lane; gi < ntok; gi += int64_t(gridDim.x) * 32) {
        const int64_t b0 = (gi / p.n) * p.n;
        float qf[HD], acc[HD];
        gload_row<HD>(p.q + gi * p.ldq + h * HD, qf, p.scale);
#pragma unroll
        for (int c = 0; c < HD; ++c) acc[c] = 0.f;
        const float2 qx = xy[gi];
        float mx = -INFINITY, l = 0.f;
        auto take = [&](float s, const __nv_bfloat16* vr) {
            if (s > mx) {
                const float c = __expf(mx - s);
                l *= c;
#pragma unroll
                for (int i = 0; i < HD; ++i) acc[i] *= c;
                mx = s;
            }
            const float e = __expf(s - mx);
            l += e;
            float vf[HD];
            gload_row<HD>(vr, vf, 1.f);
#pragma unroll
            for (int i = 0; i < HD; ++i) acc[i] = fmaf(e, vf[i], acc[i]);
        };
        const int32_t* ir = p.idx + gi * p.m;
        const uint8_t* vv = p.valid + gi * p.m;
        auto slot = [&](int32_t t) {
            const int64_t key = b0 + t;
            const float2 kx = xy[key];
            const float s = gdot<HD>(qf, p.k + key * p.ldkv + h * HD) +
                            gbias(un, p.hidden, b2, (kx.x - qx.x) * p.inv_patch, (kx.y - qx.y) * p.inv_patch);
            take(s, p.v + key * p.ldkv + h * HD);
        };
        if (p.m == 8) {  // the decoder's self_k rows: two 16-byte index loads and one 8-byte valid load
            const int4 i0 = __ldg(reinterpret_cast<const int4*>(ir)), i1 = __ldg(reinterpret_cast<const int4*>(ir) + 1);
            const uint2 vb = __ldg(reinterpret_cast<const uint2*>(vv));
            const int32_t ids[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (((j < 4 ? vb.x >> (8 * j) : vb.y >> (8 * (j - 4))) & 0xffu) != 0u) slot(ids[j]);
        } else {
            for (int j = 0; j < p.m; ++j)
                if (vv[j]) slot(ir[j]);
        }
        take(gdot<HD>(qf, p.bk + h * HD) + blank, p.bv + h * HD);
        const float il = 1.f / l;
        uint4* o = reinterpret_cast<uint4*>(out + gi * ld + h * HD);
#pragma unroll
        for (int c = 0; c < HD; c += 8) {
            uint4 w;
            __nv_bfloat162* hw = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
            for (int i = 0; i < 4; ++i) hw[i] = __floats2bfloat162_rn(acc[c + 2 * i] * il, acc[c + 2 * i + 1] * il);
            o[c / 8] = w;
        }
        lse[gi * p.heads + h] = mx + __logf(l);
    }
}

__device__ __forceinline__ float gwarp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp reduce-scatter of 32 per-lane values: returns, on lane l, the sum over the
// warp of v[l] (31 shuffles for 32 sums).  v is clobbered.
__device__ __forceinline__ float greduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? v[i] : v[i + o];
            const float keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// Backward, same layout; MW >= width bounds the per-slot register arrays.
// Per tile (32 tokens of one head) the warp's blank-k / blank-v gradients (2*HD sums) and,
// for hidden <= 8, the 4*hidden BiasNet sums are reduce-scattered so lane l keeps sum l:
// each lane writes its 32 values as one row of a per-warp 32 x 33 shared-memory tile as they
// are produced and lane l adds column l (both conflict-free); a register reduce-scatter would
// hold 32 more live values and push the thread past the 128 registers of two blocks per SM.
// G: gather mode (p.dsw set; dk / dv are formed later by the reverse-CSR gather): q and dO
// rows are dead after the scores and are re-read (L1 / L2) for the blank-row gradients, so the
// thread never holds q, dO and the dQ accumulator at once.
template <int HD, int MW, bool G>
__global__ void __launch_bounds__(256, (MW <= 8 && (HD == 16 || (HD == 32 && G))) ? 2 : 1) gattn_bwd_kernel(GAttnP p, const __nv_bfloat16* __restrict__ dout,
                                                        __nv_bfloat16* __restrict__ dq, float* __restrict__ dk,
                                                        float* __restrict__ dv, float* __restrict__ dbk,
                                                        float* __restrict__ dbv, float* __restrict__ dw1,
                                                        float* __restrict__ db1, float* __restrict__ dw2,
                                                        float* __restrict__ db2, float* __restrict__ dblank) {
    constexpr int NB = 2 * HD / 32;  // reduce-scatter rounds for the blank rows
    extern __shared__ float4 g_units[];
    gstage_units(p, g_units);
    const int lane = threadIdx.x & 31, h = threadIdx.x >> 5, H = p.hidden;
    float* rs = reinterpret_cast<float*>(g_units + p.heads * H) + h * (32 * 33);  // this warp's tile
    auto rs_sum = [&]() {  // column `lane` of the tile (after every lane wrote its row)
        __syncwarp();
        float t = 0.f;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) t += rs[r * 33 + lane];
        __syncwarp();
        return t;
    };
    const bool small_h = H <= 8;
    const float4* un = g_units + h * H;
    const float b2 = p.b2[h], blank = p.blank[h];
    const int64_t ntok = p.batch * p.n, ld = int64_t(p.heads) * HD;
    const float2* xy = reinterpret_cast<const float2*>(p.coords);
    float agx = 0.f, agy = 0.f, agb = 0.f, agw = 0.f;  // big-hidden path: lane u = unit u
    float abias = 0.f;                                 // small-hidden path: lane l = sum l of {gx, gy, gb, gw}[8]
    float ab2 = 0.f, abl = 0.f, ablk[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) ablk[r] = 0.f;
    for (int64_t base = int64_t(blockIdx.x) * 32; base < ntok; base += int64_t(gridDim.x) * 32) {
        const int64_t gi = base + lane;
        const bool act = gi < ntok;
        const int64_t row = act ? gi : base;
        const int64_t b0 = (row / p.n) * p.n;
        float qf[HD], gf[HD];
        gload_row<HD>(p.q + row * p.ldq + h * HD, qf, 1.f);
        const float2 qx = xy[row];
        float w[MW], dS[MW];
        int key[MW];  // image-local key token, -1 if none
        const int32_t* ir = p.idx + row * p.m;
        const uint8_t* vv = p.valid + row * p.m;
        float mx = -INFINITY;
        bool vec8 = false;
        int4 i0 = make_int4(0, 0, 0, 0), i1 = i0;
        uint2 vb = make_uint2(0u, 0u);
        if constexpr (MW == 8) {
            vec8 = p.m == 8;
            if (vec8) {  // the decoder's self_k rows: two 16-byte index loads, one 8-byte valid load
                i0 = __ldg(reinterpret_cast<const int4*>(ir));
                i1 = __ldg(reinterpret_cast<const int4*>(ir) + 1);
                vb = __ldg(reinterpret_cast<const uint2*>(vv));
            }
        }
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            w[j] = -INFINITY;
            key[j] = -1;
            bool ok;
            int32_t id;
            if (vec8) {
                const int4& iv = j < 4 ? i0 : i1;
                const int jj = j & 3;
                id = jj == 0 ? iv.x : jj == 1 ? iv.y : jj == 2 ? iv.z : iv.w;
                ok = act && ((j < 4 ? vb.x >> (8 * j) : vb.y >> (8 * (j - 4))) & 0xffu) != 0u;
            } else {
                ok = act && j < p.m && vv[j];
                id = ok ? ir[j] : 0;
            }
            if (ok) {
                key[j] = id;
                const float2 kx = xy[b0 + key[j]];
                w[j] = p.scale * gdot<HD>(qf, p.k + (b0 + key[j]) * p.ldkv + h * HD) +
                       gbias(un, H, b2, (kx.x - qx.x) * p.inv_patch, (kx.y - qx.y) * p.inv_patch);
                mx = fmaxf(mx, w[j]);
            }
        }
        float wb = act ? p.scale * gdot<HD>(qf, p.bk + h * HD) + blank : -INFINITY;
        mx = fmaxf(mx, wb);
        float l = 0.f;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            w[j] = key[j] >= 0 ? __expf(w[j] - mx) : 0.f;
            l += w[j];
        }
        wb = act ? __expf(wb - mx) : 0.f;
        l += wb;
        const float il = act ? 1.f / l : 0.f;
        gload_row<HD>(dout + row * ld + h * HD, gf, 1.f);
        float D = 0.f;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            w[j] *= il;
            dS[j] = key[j] >= 0 ? gdot<HD>(gf, p.v + (b0 + key[j]) * p.ldkv + h * HD) : 0.f;
            D = fmaf(w[j], dS[j], D);
        }
        wb *= il;
        const float dPb = act ? gdot<HD>(gf, p.bv + h * HD) : 0.f;
        D = fmaf(wb, dPb, D);
        const float dSb = wb * (dPb - D);
        float dqa[HD];
#pragma unroll
        for (int c = 0; c < HD; ++c) dqa[c] = 0.f;
        float s2 = 0.f;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            dS[j] = w[j] * (dS[j] - D);
            if (key[j] < 0) continue;
            s2 += dS[j];
            const int64_t kr = (b0 + key[j]) * ld + h * HD;
            const __nv_bfloat16* krow = p.k + (b0 + key[j]) * p.ldkv + h * HD;
            const float a = p.scale * dS[j];
            if (G) p.dsw[(gi * p.m + j) * p.heads + h] = make_float2(a, w[j]);
            // the key row streams through in 8-element chunks (a full row in registers would
            // double the thread's footprint and halve the resident warps)
#pragma unroll
            for (int c = 0; c < HD; c += 8) {
                const uint4 kx = __ldg(reinterpret_cast<const uint4*>(krow + c));
                const __nv_bfloat162* kh = reinterpret_cast<const __nv_bfloat162*>(&kx);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 t = __bfloat1622float2(kh[i]);
                    dqa[c + 2 * i] = fmaf(dS[j], t.x, dqa[c + 2 * i]);
                    dqa[c + 2 * i + 1] = fmaf(dS[j], t.y, dqa[c + 2 * i + 1]);
                }
                if (!G) {
#pragma unroll
                    for (int i = 0; i < 8; i += 4) {
                        gred_v4(dk + kr + c + i, a * qf[c + i], a * qf[c + i + 1], a * qf[c + i + 2],
                                a * qf[c + i + 3]);
                        gred_v4(dv + kr + c + i, w[j] * gf[c + i], w[j] * gf[c + i + 1], w[j] * gf[c + i + 2],
                                w[j] * gf[c + i + 3]);
                    }
                }
            }
        }
        if (act) {
            float bkf[HD];
            gload_row<HD>(p.bk + h * HD, bkf, 1.f);  // uniform across the warp: one broadcast line
            uint4* o = reinterpret_cast<uint4*>(dq + gi * p.ldd + h * HD);
#pragma unroll
            for (int c = 0; c < HD; c += 8) {
                uint4 v;
                __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    hv[i] = __floats2bfloat162_rn(p.scale * fmaf(dSb, bkf[c + 2 * i], dqa[c + 2 * i]),
                                                  p.scale * fmaf(dSb, bkf[c + 2 * i + 1], dqa[c + 2 * i + 1]));
                o[c / 8] = v;
            }
            ab2 += s2;
            abl += dSb;
        }
        // blank rows: values {scale dSb q[c]} then {wb g[c]}, 32 per round
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            if (G) {
                // re-read q / dO in 8-element chunks (dead registers since the scores)
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    const int e = r * 32 + i;
                    const __nv_bfloat16* src = e < HD ? p.q + row * p.ldq + h * HD + e : dout + row * ld + h * HD + (e - HD);
                    const float mul = e < HD ? p.scale * dSb : wb;
                    const uint4 x = __ldg(reinterpret_cast<const uint4*>(src));
                    const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float2 f = __bfloat1622float2(xh[t]);
                        rs[lane * 33 + i + 2 * t] = mul * f.x;
                        rs[lane * 33 + i + 2 * t + 1] = mul * f.y;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int e = r * 32 + i;
                    rs[lane * 33 + i] = e < HD ? p.scale * dSb * qf[e] : wb * gf[e - HD];
                }
            }
            ablk[r] += rs_sum();
        }
        // BiasNet gradients of the tile's pairs
        if (small_h) {
            float* v = rs + lane * 33;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float gx = 0.f, gy = 0.f, gb = 0.f, gw = 0.f;
                if (u < H) {
                    const float4 wu = un[u];
#pragma unroll
                    for (int j = 0; j < MW; ++j) {
                        if (key[j] < 0) continue;
                        const float2 kx = xy[b0 + key[j]];
                        const float ox = (kx.x - qx.x) * p.inv_patch, oy = (kx.y - qx.y) * p.inv_patch;
                        const float th = tanh_fast(fmaf(wu.x, ox, fmaf(wu.y, oy, wu.z)));
                        const float dpre = dS[j] * wu.w * (1.f - th * th);
                        gx = fmaf(dpre, ox, gx);
                        gy = fmaf(dpre, oy, gy);
                        gb += dpre;
                        gw = fmaf(dS[j], th, gw);
                    }
                }
                v[u] = gx;
                v[8 + u] = gy;
                v[16 + u] = gb;
                v[24 + u] = gw;
            }
            abias += rs_sum();
        } else {
            for (int u = 0; u < H; ++u) {
                const float4 wu = un[u];
                float gx = 0.f, gy = 0.f, gb = 0.f, gw = 0.f;
#pragma unroll
                for (int j = 0; j < MW; ++j) {
                    if (key[j] < 0) continue;
                    const float2 kx = xy[b0 + key[j]];
                    const float ox = (kx.x - qx.x) * p.inv_patch, oy = (kx.y - qx.y) * p.inv_patch;
                    const float th = tanh_fast(fmaf(wu.x, ox, fmaf(wu.y, oy, wu.z)));
                    const float dpre = dS[j] * wu.w * (1.f - th * th);
                    gx = fmaf(dpre, ox, gx);
                    gy = fmaf(dpre, oy, gy);
                    gb += dpre;
                    gw = fmaf(dS[j], th, gw);
                }
                gx = gwarp_sum(gx);
                gy = gwarp_sum(gy);
                gb = gwarp_sum(gb);
                gw = gwarp_sum(gw);
                if (lane == u) {
                    agx += gx;
                    agy += gy;
                    agb += gb;
                    agw += gw;
                }
            }
        }
    }
    if (small_h) {
        const int u = lane & 7, kind = lane >> 3;
        if (u < H) {
            float* dst = kind == 0 ? dw1 + h * 2 * H + u
                       : kind == 1 ? dw1 + h * 2 * H + H + u
                       : kind == 2 ? db1 + h * H + u
                                   : dw2 + h * H + u;
            atomicAdd(dst, abias);
        }
    } else if (lane < H) {
        atomicAdd(dw1 + h * 2 * H + lane, agx);
        atomicAdd(dw1 + h * 2 * H + H + lane, agy);
        atomicAdd(db1 + h * H + lane, agb);
        atomicAdd(dw2 + h * H + lane, agw);
    }
    ab2 = gwarp_sum(ab2);
    abl = gwarp_sum(abl);
    if (lane == 0) {
        atomicAdd(db2 + h, ab2);
        atomicAdd(dblank + h, abl);
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        const int e = r * 32 + lane;
        atomicAdd(e < HD ? dbk + h * HD + e : dbv + h * HD + (e - HD), ablk[r]);
    }
}

// ------------------------------------------------------------ row-parallel kernels
// Warp per query, lanes over the D = heads*HD row (VPL = D/32 contiguous dims per lane,
// LPH = 32/heads lanes per head): every q / k / v / dO row is read as ONE coalesced
// D*2-byte transaction by the warp instead of 2*HD-byte segments per (token, head) thread,
// so the L1 wavefronts per byte drop by 8x at D = 256 -- the thread-per-(token, head) kernels
// above were L1-throughput bound (87 %).  Scores: per-lane partial dot products (+ the lane's
// share of the BiasNet hidden units) reduced over the head's LPH lanes.
template <int VPL>
__device__ __forceinline__ void ld_slice(const __nv_bfloat16* p, uint32_t (&w)[VPL / 2]) {
    if constexpr (VPL == 2) {
        w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
    } else if constexpr (VPL == 4) {
        const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = x.x;
        w[1] = x.y;
    } else {
#pragma unroll
        for (int c = 0; c < VPL / 8; ++c) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(p) + c);
            w[4 * c] = x.x;
            w[4 * c + 1] = x.y;
            w[4 * c + 2] = x.z;
            w[4 * c + 3] = x.w;
        }
    }
}
template <int VPL>
__device__ __forceinline__ void unpack_slice(const uint32_t (&w)[VPL / 2], float (&f)[VPL], float mul) {
#pragma unroll
    for (int i = 0; i < VPL / 2; ++i) {
        const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        f[2 * i] = t.x * mul;
        f[2 * i + 1] = t.y * mul;
    }
}
template <int VPL>
__device__ __forceinline__ float dot_slice(const float (&a)[VPL], const uint32_t (&w)[VPL / 2]) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPL / 2; ++i) {
        const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        s = fmaf(a[2 * i], t.x, fmaf(a[2 * i + 1], t.y, s));
    }
    return s;
}
template <int VPL>
__device__ __forceinline__ void st_slice(__nv_bfloat16* p, const float (&f)[VPL], float mul) {
    uint32_t w[VPL / 2];
#pragma unroll
    for (int i = 0; i < VPL / 2; ++i) {
        const __nv_bfloat162 t = __floats2bfloat162_rn(f[2 * i] * mul, f[2 * i + 1] * mul);
        w[i] = *reinterpret_cast<const uint32_t*>(&t);
    }
    if constexpr (VPL == 2) {
        *reinterpret_cast<unsigned*>(p) = w[0];
    } else if constexpr (VPL == 4) {
        *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    } else {
#pragma unroll
        for (int c = 0; c < VPL / 8; ++c)
            reinterpret_cast<uint4*>(p)[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    }
}
// sum over the LPH lanes of a head (xor butterfly: every lane of the group gets the same bits)
__device__ __forceinline__ float group_sum(float v, int lph) {
    for (int o = lph >> 1; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// neighbour ids / valid flags of row gi (two 16-byte + one 8-byte load for the decoder's 8-wide rows)
template <int MW>
__device__ __forceinline__ void row_ids(const GAttnP& p, int64_t gi, int (&key)[MW]) {
    const int32_t* ir = p.idx + gi * p.m;
    const uint8_t* vv = p.valid + gi * p.m;
    if (MW == 8 && p.m == 8) {
        const int4 i0 = __ldg(reinterpret_cast<const int4*>(ir)), i1 = __ldg(reinterpret_cast<const int4*>(ir) + 1);
        const uint2 vb = __ldg(reinterpret_cast<const uint2*>(vv));
        const int ids[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
        for (int j = 0; j < MW; ++j)
            key[j] = ((j < 4 ? vb.x >> (8 * j) : vb.y >> (8 * (j - 4))) & 0xffu) ? ids[j & 7] : -1;
    } else {
#pragma unroll
        for (int j = 0; j < MW; ++j) key[j] = (j < p.m && __ldg(vv + j)) ? __ldg(ir + j) : -1;
    }
}

// Register variant for the wide (8-slot) rows: the k AND v row slices of all slots are loaded
// up front (one memory round trip per query) and held in registers -- at 128 registers two
// 256-thread blocks fit an SM, which beats the shared-memory-staged pipeline (one block of
// eight warps) on these latency-bound rows.
template <int VPL, int MW>
__global__ void __launch_bounds__(256, 2) gattn_fwd_reg_kernel(GAttnP p, __nv_bfloat16* __restrict__ out,
                                                               float* __restrict__ lse) {
    constexpr int D = 32 * VPL;
    extern __shared__ float4 g_units[];
    gstage_units(p, g_units);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = p.heads, lph = 32 / H, h = lane / lph, sub = lane - h * lph, hid = p.hidden;
    const float4* un = g_units + h * hid;
    const float b2 = p.b2[h], blank = p.blank[h];
    const int64_t ntok = p.batch * p.n, nw = int64_t(gridDim.x) * 8;
    const float2* xy = reinterpret_cast<const float2*>(p.coords);
    uint32_t bkw[VPL / 2], bvw[VPL / 2];
    ld_slice<VPL>(p.bk + lane * VPL, bkw);
    ld_slice<VPL>(p.bv + lane * VPL, bvw);
    for (int64_t gi = int64_t(blockIdx.x) * 8 + warp; gi < ntok; gi += nw) {
        const int64_t b0 = (gi / p.n) * p.n;
        int key[MW];
        row_ids<MW>(p, gi, key);
        uint32_t qw[VPL / 2];
        ld_slice<VPL>(p.q + gi * p.ldq + lane * VPL, qw);
        uint32_t kw[MW][VPL / 2], vw[MW][VPL / 2];
#pragma unroll
        for (int j = 0; j < MW; ++j)
            if (key[j] >= 0) {
                ld_slice<VPL>(p.k + (b0 + key[j]) * p.ldkv + lane * VPL, kw[j]);
                ld_slice<VPL>(p.v + (b0 + key[j]) * p.ldkv + lane * VPL, vw[j]);
            }
        float qf[VPL];
        unpack_slice<VPL>(qw, qf, p.scale);
        const float2 qx = xy[gi];
        float s[MW];
        const float sb = group_sum(dot_slice<VPL>(qf, bkw), lph) + blank;
        float mx = sb;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            s[j] = -INFINITY;
            if (key[j] < 0) continue;  // warp-uniform
            const float2 kx = xy[b0 + key[j]];
            const float ox = (kx.x - qx.x) * p.inv_patch, oy = (kx.y - qx.y) * p.inv_patch;
            float part = dot_slice<VPL>(qf, kw[j]);
            for (int u = sub; u < hid; u += lph) {
                const float4 w = un[u];
                part = fmaf(w.w, tanh_fast(fmaf(w.x, ox, fmaf(w.y, oy, w.z))), part);
            }
            s[j] = group_sum(part, lph) + b2;
            mx = fmaxf(mx, s[j]);
        }
        float acc[VPL];
        const float pb = __expf(sb - mx);
        float l = pb;
        unpack_slice<VPL>(bvw, acc, pb);
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            if (key[j] < 0) continue;
            const float e = __expf(s[j] - mx);
            l += e;
#pragma unroll
            for (int i = 0; i < VPL / 2; ++i) {
                const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vw[j][i]));
                acc[2 * i] = fmaf(e, t.x, acc[2 * i]);
                acc[2 * i + 1] = fmaf(e, t.y, acc[2 * i + 1]);
            }
        }
        st_slice<VPL>(out + gi * D + lane * VPL, acc, 1.f / l);
        if (sub == 0) lse[gi * H + h] = mx + __logf(l);
    }
}

// cp.async of the lane's VPL-element slice of one row into shared memory
template <int VPL>
__device__ __forceinline__ void cp_slice(__nv_bfloat16* dst, const __nv_bfloat16* src) {
    const uint32_t d = smem_u32(dst);
    if constexpr (VPL == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
    } else if constexpr (VPL == 4) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
    } else {
#pragma unroll
        for (int c = 0; c < VPL / 8; ++c)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + 16 * c), "l"(src + 8 * c)
                         : "memory");
    }
}
template <int VPL>
__device__ __forceinline__ void lds_slice(const __nv_bfloat16* p, uint32_t (&w)[VPL / 2]) {
    if constexpr (VPL == 2) {
        w[0] = *reinterpret_cast<const unsigned*>(p);
    } else if constexpr (VPL == 4) {
        const uint2 x = *reinterpret_cast<const uint2*>(p);
        w[0] = x.x;
        w[1] = x.y;
    } else {
#pragma unroll
        for (int c = 0; c < VPL / 8; ++c) {
            const uint4 x = reinterpret_cast<const uint4*>(p)[c];
            w[4 * c] = x.x;
            w[4 * c + 1] = x.y;
            w[4 * c + 2] = x.z;
            w[4 * c + 3] = x.w;
        }
    }
}

// One pipeline stage of a warp: NR rows of D bf16 (q, [dO,] k_0..k_{MW-1}, v_0..v_{MW-1}) and
// the coordinates of the query (slot 0) and its neighbours (slots 1..MW).
template <int VPL, int MW, bool BWD>
struct GStage {
    static constexpr int D = 32 * VPL;
    static constexpr int NR = (BWD ? 2 : 1) + 2 * MW;
    static constexpr int KR = BWD ? 2 : 1;  // first key row
    static constexpr int VR = KR + MW;      // first value row
    static constexpr size_t ROW_BYTES = size_t(NR) * D * 2;
    static constexpr size_t BYTES = (ROW_BYTES + size_t(MW + 1) * 8 + 15) / 16 * 16;
};
template <int VPL>
constexpr int g_warps() { return VPL >= 16 ? 4 : 8; }  // <= ~150 KB of stages per block

// Issue the rows of query gi (neighbour ids in key[]) into stage `st`.
template <int VPL, int MW, bool BWD>
__device__ __forceinline__ void g_issue(uint8_t* st, const GAttnP& p, const __nv_bfloat16* dout, int64_t gi,
                                        int64_t b0, const int (&key)[MW], int lane) {
    using G = GStage<VPL, MW, BWD>;
    constexpr int D = G::D;
    auto* rows = reinterpret_cast<__nv_bfloat16*>(st) + lane * VPL;
    cp_slice<VPL>(rows, p.q + gi * p.ldq + lane * VPL);
    if constexpr (BWD) cp_slice<VPL>(rows + D, dout + gi * D + lane * VPL);
#pragma unroll
    for (int j = 0; j < MW; ++j)
        if (key[j] >= 0) {
            cp_slice<VPL>(rows + (G::KR + j) * D, p.k + (b0 + key[j]) * p.ldkv + lane * VPL);
            cp_slice<VPL>(rows + (G::VR + j) * D, p.v + (b0 + key[j]) * p.ldkv + lane * VPL);
        }
    // coordinates: lane 0 the query's, lane 1 + j neighbour j's
    float2* cx = reinterpret_cast<float2*>(st + G::ROW_BYTES);
    int64_t src = lane == 0 ? gi : -1;
#pragma unroll
    for (int j = 0; j < MW; ++j)
        if (lane == j + 1 && key[j] >= 0) src = b0 + key[j];
    if (src >= 0)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(cx + lane)),
                     "l"(reinterpret_cast<const float2*>(p.coords) + src)
                     : "memory");
}

template <int VPL, int MW>
__global__ void __launch_bounds__(256) gattn_fwd_row_kernel(GAttnP p, __nv_bfloat16* __restrict__ out,
                                                             float* __restrict__ lse) {
    using G = GStage<VPL, MW, false>;
    constexpr int D = G::D;
    extern __shared__ float4 g_units[];
    gstage_units(p, g_units);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int H = p.heads, lph = 32 / H, h = lane / lph, sub = lane - h * lph, hid = p.hidden;
    const float4* un = g_units + h * hid;
    uint8_t* ring = reinterpret_cast<uint8_t*>(g_units + H * hid) + size_t(warp) * 2 * G::BYTES;
    const float b2 = p.b2[h], blank = p.blank[h];
    const int64_t ntok = p.batch * p.n, nw = int64_t(gridDim.x) * nwb;
    uint32_t bkw[VPL / 2], bvw[VPL / 2];
    ld_slice<VPL>(p.bk + lane * VPL, bkw);
    ld_slice<VPL>(p.bv + lane * VPL, bvw);
    int64_t gi = int64_t(blockIdx.x) * nwb + warp;
    int key0[MW], key1[MW];
    if (gi < ntok) {
        row_ids<MW>(p, gi, key0);
        g_issue<VPL, MW, false>(ring, p, nullptr, gi, (gi / p.n) * p.n, key0, lane);
    }
    cp_async_commit();
    if (gi + nw < ntok) row_ids<MW>(p, gi + nw, key1);
    for (int it = 0; gi < ntok; gi += nw, ++it) {
        uint8_t* cur = ring + (it & 1) * G::BYTES;
        const int64_t g1 = gi + nw;
        if (g1 < ntok) g_issue<VPL, MW, false>(ring + ((it + 1) & 1) * G::BYTES, p, nullptr, g1, (g1 / p.n) * p.n, key1, lane);
        cp_async_commit();
        int key2[MW];
        if (g1 + nw < ntok) row_ids<MW>(p, g1 + nw, key2);
        cp_async_wait<1>();
        __syncwarp();
        const __nv_bfloat16* rows = reinterpret_cast<const __nv_bfloat16*>(cur) + lane * VPL;
        const float2* cx = reinterpret_cast<const float2*>(cur + G::ROW_BYTES);
        uint32_t qw[VPL / 2];
        lds_slice<VPL>(rows, qw);
        float qf[VPL];
        unpack_slice<VPL>(qw, qf, p.scale);
        const float2 qx = cx[0];
        float s[MW];
        const float sb = group_sum(dot_slice<VPL>(qf, bkw), lph) + blank;
        float mx = sb;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            s[j] = -INFINITY;
            if (key0[j] < 0) continue;  // warp-uniform
            uint32_t kw[VPL / 2];
            lds_slice<VPL>(rows + (G::KR + j) * D, kw);
            const float2 kx = cx[1 + j];
            const float ox = (kx.x - qx.x) * p.inv_patch, oy = (kx.y - qx.y) * p.inv_patch;
            float part = dot_slice<VPL>(qf, kw);
            for (int u = sub; u < hid; u += lph) {
                const float4 w = un[u];
                part = fmaf(w.w, tanh_fast(fmaf(w.x, ox, fmaf(w.y, oy, w.z))), part);
            }
            s[j] = group_sum(part, lph) + b2;
            mx = fmaxf(mx, s[j]);
        }
        float acc[VPL];
        const float pb = __expf(sb - mx);
        float l = pb;
        unpack_slice<VPL>(bvw, acc, pb);
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            if (key0[j] < 0) continue;
            uint32_t vw[VPL / 2];
            lds_slice<VPL>(rows + (G::VR + j) * D, vw);
            const float e = __expf(s[j] - mx);
            l += e;
#pragma unroll
            for (int i = 0; i < VPL / 2; ++i) {
                const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vw[i]));
                acc[2 * i] = fmaf(e, t.x, acc[2 * i]);
                acc[2 * i + 1] = fmaf(e, t.y, acc[2 * i + 1]);
            }
        }
        st_slice<VPL>(out + gi * D + lane * VPL, acc, 1.f / l);
        if (sub == 0) lse[gi * H + h] = mx + __logf(l);
        __syncwarp();  // stage consumed before it is refilled
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            key0[j] = key1[j];
            key1[j] = key2[j];
        }
    }
    cp_async_wait<0>();
}

// Backward, same staging.  dk / dv: gather mode writes {scale dS, P} per (entry, head) for
// gattn_kv_gather_kernel; one-to-one mode (p.o2o: the only key of row i is token i) stores
// bf16 dk / dv rows directly; otherwise coalesced 16-byte fp32 reductions per row.
// Parameter gradients accumulate per lane (blank rows: the lane's dims; BiasNet: the lane's
// hidden units u = sub + t*LPH), then per block in shared memory, then one atomic each.
template <int VPL, int MW, int UPL>
__global__ void __launch_bounds__(256) gattn_bwd_row_kernel(GAttnP p, const __nv_bfloat16* __restrict__ dout,
                                                             __nv_bfloat16* __restrict__ dq, float* __restrict__ dk,
                                                             float* __restrict__ dv, float* __restrict__ dbk,
                                                             float* __restrict__ dbv, float* __restrict__ dw1,
                                                             float* __restrict__ db1, float* __restrict__ dw2,
                                                             float* __restrict__ db2, float* __restrict__ dblank) {
    using G = GStage<VPL, MW, true>;
    constexpr int D = G::D;
    extern __shared__ float4 g_units[];
    gstage_units(p, g_units);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int H = p.heads, lph = 32 / H, h = lane / lph, sub = lane - h * lph, hid = p.hidden;
    const float4* un = g_units + h * hid;
    uint8_t* ring = reinterpret_cast<uint8_t*>(g_units + H * hid) + size_t(warp) * 2 * G::BYTES;
    const float b2 = p.b2[h], blank = p.blank[h];
    const int64_t ntok = p.batch * p.n, nw = int64_t(gridDim.x) * nwb;
    uint32_t bkw[VPL / 2], bvw[VPL / 2];
    ld_slice<VPL>(p.bk + lane * VPL, bkw);
    ld_slice<VPL>(p.bv + lane * VPL, bvw);
    float abk[VPL], abv[VPL], ag[UPL][4], ab2 = 0.f, abl = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) abk[i] = abv[i] = 0.f;
#pragma unroll
    for (int t = 0; t < UPL; ++t) ag[t][0] = ag[t][1] = ag[t][2] = ag[t][3] = 0.f;
    int64_t gi = int64_t(blockIdx.x) * nwb + warp;
    int key0[MW], key1[MW];
    if (gi < ntok) {
        row_ids<MW>(p, gi, key0);
        g_issue<VPL, MW, true>(ring, p, dout, gi, (gi / p.n) * p.n, key0, lane);
    }
    cp_async_commit();
    if (gi + nw < ntok) row_ids<MW>(p, gi + nw, key1);
    for (int it = 0; gi < ntok; gi += nw, ++it) {
        uint8_t* cur = ring + (it & 1) * G::BYTES;
        const int64_t g1 = gi + nw;
        if (g1 < ntok) g_issue<VPL, MW, true>(ring + ((it + 1) & 1) * G::BYTES, p, dout, g1, (g1 / p.n) * p.n, key1, lane);
        cp_async_commit();
        int key2[MW];
        if (g1 + nw < ntok) row_ids<MW>(p, g1 + nw, key2);
        cp_async_wait<1>();
        __syncwarp();
        const int64_t b0 = (gi / p.n) * p.n;
        const __nv_bfloat16* rows = reinterpret_cast<const __nv_bfloat16*>(cur) + lane * VPL;
        const float2* cx = reinterpret_cast<const float2*>(cur + G::ROW_BYTES);
        float qf[VPL], gf[VPL];
        {
            uint32_t w[VPL / 2];
            lds_slice<VPL>(rows, w);
            unpack_slice<VPL>(w, qf, 1.f);
            lds_slice<VPL>(rows + D, w);
            unpack_slice<VPL>(w, gf, 1.f);
        }
        const float2 qx = cx[0];
        float s[MW];
        const float sb = p.scale * group_sum(dot_slice<VPL>(qf, bkw), lph) + blank;
        float mx = sb;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            s[j] = -INFINITY;
            if (key0[j] < 0) continue;
            uint32_t kw[VPL / 2];
            lds_slice<VPL>(rows + (G::KR + j) * D, kw);
            const float2 kx = cx[1 + j];
            const float ox = (kx.x - qx.x) * p.inv_patch, oy = (kx.y - qx.y) * p.inv_patch;
            float part = p.scale * dot_slice<VPL>(qf, kw);
            for (int u = sub; u < hid; u += lph) {
                const float4 w = un[u];
                part = fmaf(w.w, tanh_fast(fmaf(w.x, ox, fmaf(w.y, oy, w.z))), part);
            }
            s[j] = group_sum(part, lph) + b2;
            mx = fmaxf(mx, s[j]);
        }
        float pb = __expf(sb - mx), l = pb;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            s[j] = key0[j] >= 0 ? __expf(s[j] - mx) : 0.f;
            l += s[j];
        }
        const float il = 1.f / l;
        pb *= il;
        const float dPb = group_sum(dot_slice<VPL>(gf, bvw), lph);
        float Dsum = pb * dPb, dS[MW];
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            s[j] *= il;
            dS[j] = 0.f;
            if (key0[j] < 0) continue;
            uint32_t vw[VPL / 2];
            lds_slice<VPL>(rows + (G::VR + j) * D, vw);
            dS[j] = group_sum(dot_slice<VPL>(gf, vw), lph);
            Dsum = fmaf(s[j], dS[j], Dsum);
        }
        const float dSb = pb * (dPb - Dsum);
        float dqa[VPL];
        unpack_slice<VPL>(bkw, dqa, dSb);
        float s2 = 0.f;
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            if (key0[j] < 0) continue;
            dS[j] = s[j] * (dS[j] - Dsum);
            s2 += dS[j];
            float kf[VPL];
            {
                uint32_t kw[VPL / 2];
                lds_slice<VPL>(rows + (G::KR + j) * D, kw);
                unpack_slice<VPL>(kw, kf, 1.f);
            }
#pragma unroll
            for (int i = 0; i < VPL; ++i) dqa[i] = fmaf(dS[j], kf[i], dqa[i]);
            const float a = p.scale * dS[j];
            if (p.dsw) {
                if (sub == 0) p.dsw[(gi * p.m + j) * H + h] = make_float2(a, s[j]);
            } else if (p.o2o) {  // MW == 1: the key row is row gi
                float t[VPL];
#pragma unroll
                for (int i = 0; i < VPL; ++i) t[i] = a * qf[i];
                st_slice<VPL>(reinterpret_cast<__nv_bfloat16*>(dk) + gi * p.lddkv + lane * VPL, t, 1.f);
                st_slice<VPL>(reinterpret_cast<__nv_bfloat16*>(dv) + gi * p.lddkv + lane * VPL, gf, s[j]);
            } else {
                float* pk = dk + (b0 + key0[j]) * D + lane * VPL;
                float* pv = dv + (b0 + key0[j]) * D + lane * VPL;
#pragma unroll
                for (int i = 0; i < VPL; i += 2) {
                    if constexpr (VPL % 4 == 0) {
                        if (i % 4 == 0) {
                            gred_v4(pk + i, a * qf[i], a * qf[i + 1], a * qf[i + 2], a * qf[i + 3]);
                            gred_v4(pv + i, s[j] * gf[i], s[j] * gf[i + 1], s[j] * gf[i + 2], s[j] * gf[i + 3]);
                        }
                    } else {
                        atomicAdd(pk + i, a * qf[i]);
                        atomicAdd(pk + i + 1, a * qf[i + 1]);
                        atomicAdd(pv + i, s[j] * gf[i]);
                        atomicAdd(pv + i + 1, s[j] * gf[i + 1]);
                    }
                }
            }
        }
        if (p.o2o && key0[0] < 0) {  // an invalid one-to-one row still owns its dk / dv rows
            float z[VPL];
#pragma unroll
            for (int i = 0; i < VPL; ++i) z[i] = 0.f;
            st_slice<VPL>(reinterpret_cast<__nv_bfloat16*>(dk) + gi * p.lddkv + lane * VPL, z, 1.f);
            st_slice<VPL>(reinterpret_cast<__nv_bfloat16*>(dv) + gi * p.lddkv + lane * VPL, z, 1.f);
        }
        st_slice<VPL>(dq + gi * p.ldd + lane * VPL, dqa, p.scale);
        // parameter gradients
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            abk[i] = fmaf(p.scale * dSb, qf[i], abk[i]);
            abv[i] = fmaf(pb, gf[i], abv[i]);
        }
        if (sub == 0) {
            ab2 += s2;
            abl += dSb;
        }
#pragma unroll
        for (int t = 0; t < UPL; ++t) {
            const int u = sub + t * lph;
            if (u >= hid) break;
            const float4 w = un[u];
#pragma unroll
            for (int j = 0; j < MW; ++j) {
                if (key0[j] < 0) continue;
                const float2 kx = cx[1 + j];
                const float ox = (kx.x - qx.x) * p.inv_patch, oy = (kx.y - qx.y) * p.inv_patch;
                const float th = tanh_fast(fmaf(w.x, ox, fmaf(w.y, oy, w.z)));
                const float dpre = dS[j] * w.w * (1.f - th * th);
                ag[t][0] = fmaf(dpre, ox, ag[t][0]);
                ag[t][1] = fmaf(dpre, oy, ag[t][1]);
                ag[t][2] += dpre;
                ag[t][3] = fmaf(dS[j], th, ag[t][3]);
            }
        }
        __syncwarp();  // stage consumed before it is refilled
#pragma unroll
        for (int j = 0; j < MW; ++j) {
            key0[j] = key1[j];
            key1[j] = key2[j];
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // every warp done with its stages: the ring becomes the reduction buffer
    // block reduction: per-warp rows [D] dbk | [D] dbv | [H][hid][4] BiasNet | [H] db2 | [H] dblank
    float* red = reinterpret_cast<float*>(g_units + H * hid);
    const int W = 2 * D + 4 * H * hid + 2 * H;
    float* mine = red + warp * W;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
        mine[lane * VPL + i] = abk[i];
        mine[D + lane * VPL + i] = abv[i];
    }
#pragma unroll
    for (int t = 0; t < UPL; ++t) {
        const int u = sub + t * lph;
        if (u < hid)
#pragma unroll
            for (int c = 0; c < 4; ++c) mine[2 * D + (h * hid + u) * 4 + c] = ag[t][c];
    }
    if (sub == 0) {
        mine[2 * D + 4 * H * hid + h] = ab2;
        mine[2 * D + 4 * H * hid + H + h] = abl;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < W; e += blockDim.x) {
        float v = 0.f;
        for (int w = 0; w < nwb; ++w) v += red[w * W + e];
        if (p.part) p.part[size_t(blockIdx.x) * W + e] = v;
        else atomicAdd(grad_dst(e, D, H, hid, dbk, dbv, dw1, db1, dw2, db2, dblank), v);
    }
}

void rev_csr_build(const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t nq, int64_t nk, int k,
                   int32_t* off, int32_t* cur, int32_t* ent, int32_t* ent_key, cudaStream_t st);

// dk / dv by gathering over the key-sorted reverse CSR of the rows (the interpolation
// backward's balanced scheme, interp.cu): warps walk chunks of 32 entries, lanes over the
// D = heads*HD row (VPL dims each, inside one head), flush per key change.
template <int D>
__global__ void __launch_bounds__(256) gattn_kv_gather_kernel(const int32_t* __restrict__ off,
                                                              const int32_t* __restrict__ ent,
                                                              const int32_t* __restrict__ ent_key,
                                                              const float2* __restrict__ dsw, int64_t batch,
                                                              int64_t n, int m, int heads, int hd,
                                                              const __nv_bfloat16* __restrict__ q, int64_t ldq,
                                                              const __nv_bfloat16* __restrict__ dout,
                                                              float* __restrict__ dk, float* __restrict__ dv) {
    constexpr int VPL = D / 32;
    const int lane = threadIdx.x & 31, h = lane * VPL / hd;
    const int64_t span = n * m, total = batch * span, nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
    float ak[VPL], av[VPL];
    auto flush = [&](int32_t key) {
        float* pk = dk + int64_t(key) * D + lane * VPL;
        float* pv = dv + int64_t(key) * D + lane * VPL;
        if constexpr (VPL % 4 == 0) {
#pragma unroll
            for (int c = 0; c < VPL; c += 4) {
                gred_v4(pk + c, ak[c], ak[c + 1], ak[c + 2], ak[c + 3]);
                gred_v4(pv + c, av[c], av[c + 1], av[c + 2], av[c + 3]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < VPL; ++c) {
                atomicAdd(pk + c, ak[c]);
                atomicAdd(pv + c, av[c]);
            }
        }
#pragma unroll
        for (int i = 0; i < VPL; ++i) ak[i] = av[i] = 0.f;
    };
    for (int64_t c0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; c0 < total; c0 += nwarps * 32) {
        const int64_t pos = c0 + lane;
        int32_t mkey = -1, me = 0;
        if (pos < total) {
            const int64_t b = pos / span;
            if (pos - b * span < off[b * (n + 1) + n]) {
                me = __ldg(ent + pos);
                mkey = __ldg(ent_key + pos);
            }
        }
        if (__ballot_sync(0xffffffffu, mkey >= 0) == 0u) continue;
#pragma unroll
        for (int i = 0; i < VPL; ++i) ak[i] = av[i] = 0.f;
        int32_t cur = -1;
#pragma unroll 4
        for (int u = 0; u < 32; ++u) {
            const int32_t key = __shfl_sync(0xffffffffu, mkey, u);
            const int32_t e = __shfl_sync(0xffffffffu, me, u);
            if (key < 0) continue;  // uniform
            if (key != cur) {
                if (cur >= 0) flush(cur);
                cur = key;
            }
            const float2 sw = __ldg(dsw + int64_t(e) * heads + h);
            const int64_t row = e / m;
            const __nv_bfloat16* qr = q + row * ldq + lane * VPL;
            const __nv_bfloat16* gr = dout + row * D + lane * VPL;
            if constexpr (VPL == 1) {
                ak[0] = fmaf(sw.x, __bfloat162float(qr[0]), ak[0]);
                av[0] = fmaf(sw.y, __bfloat162float(gr[0]), av[0]);
            } else {
#pragma unroll
                for (int c = 0; c < VPL; c += 2) {
                    const float2 tq = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qr + c));
                    const float2 tg = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(gr + c));
                    ak[c] = fmaf(sw.x, tq.x, ak[c]);
                    ak[c + 1] = fmaf(sw.x, tq.y, ak[c + 1]);
                    av[c] = fmaf(sw.y, tg.x, av[c]);
                    av[c + 1] = fmaf(sw.y, tg.y, av[c + 1]);
                }
            }
        }
        if (cur >= 0) flush(cur);
    }
}

static bool gattn_gather_ok(const affmae_attn_desc* a) {
    const int d = a->heads * a->head_dim;
    return d == 32 || d == 64 || d == 128 || d == 256 || d == 512;
}

size_t gattn_bwd_workspace(const affmae_attn_desc* a, int64_t batch, int64_t tokens, int64_t width) {
    if (!a || !gattn_gather_ok(a)) return 0;
    const int64_t ents = batch * tokens * width;
    return size_t(batch * (tokens + 1) + batch * tokens + 2 * ents) * 4 + size_t(ents) * a->heads * 8 + 1024;
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
    if (a->heads > kGMaxHeads) return fail(AFFMAE_EUNSUPPORTED, "gattn: at most 8 heads");
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
    p.ldq = p.ldkv = p.ldd = p.lddkv = int64_t(a->heads) * a->head_dim;
    return AFFMAE_OK;
}
// optional strides (0 = dense); row starts stay 16-byte aligned for the vector row loads
static int gattn_strides(GAttnP& p, int64_t ldq, int64_t ldkv, int64_t ldd, int64_t lddkv) {
    const int64_t D = p.ldq;
    for (int64_t* f : {&ldq, &ldkv, &ldd, &lddkv}) {
        if (*f == 0) *f = D;
        if (*f < D || *f % 8) return fail(AFFMAE_ECONFIG, "gattn: row stride below D or not a multiple of 8");
    }
    p.ldq = ldq;
    p.ldkv = ldkv;
    p.ldd = ldd;
    p.lddkv = lddkv;
    return AFFMAE_OK;
}

static unsigned gattn_blocks(int64_t tokens, int heads, int per_sm_threads) {
    const int64_t tiles = (tokens + 31) / 32;
    const int64_t resident = std::max<int64_t>(1, per_sm_threads / (32 * heads)) * kNumSMs;
    return unsigned(std::max<int64_t>(1, std::min(tiles, resident)));
}

// Row kernels cover D = 32*VPL, VPL in {2, 4, 8, 16}, heads | 32, width <= 8, hidden <= 8*LPH.
static int row_vpl(const affmae_attn_desc* a, int64_t width) {
    const int D = a->heads * a->head_dim;
    if (width > 8 || 32 % a->heads != 0 || D % 32 != 0) return 0;
    const int vpl = D / 32;
    if (vpl != 2 && vpl != 4 && vpl != 8 && vpl != 16) return 0;
    if (a->bias_hidden > 8 * (32 / a->heads)) return 0;
    return vpl;
}

template <int VPL, int MW, bool BWD>
static size_t row_smem(const GAttnP& p) {
    const size_t units = size_t(p.heads) * p.hidden * sizeof(float4);
    size_t ring = size_t(g_warps<VPL>()) * 2 * GStage<VPL, MW, BWD>::BYTES;
    if (BWD) ring = std::max(ring, size_t(g_warps<VPL>()) * (2 * 32 * VPL + 4 * p.heads * p.hidden + 2 * p.heads) * 4);
    return units + ring;
}
template <typename K>
static int row_grid(K kern, size_t smem, int warps, int64_t tokens, unsigned& blocks) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return cuda_status(e, "gattn: cudaFuncSetAttribute");
    }
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * warps, smem);
    if (e != cudaSuccess) return cuda_status(e, "gattn: occupancy");
    if (occ < 1) return fail(AFFMAE_EUNSUPPORTED, "gattn: row kernel does not fit on an SM");
    const int64_t want = (tokens + warps - 1) / warps;
    blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(occ) * device_sms())));
    return AFFMAE_OK;
}

template <int VPL, int MW>
static int row_fwd_launch2(const GAttnP& p, __nv_bfloat16* o, float* lse, cudaStream_t st) {
    auto k = gattn_fwd_row_kernel<VPL, MW>;
    const size_t sm = row_smem<VPL, MW, false>(p);
    unsigned nb = 0;
    if (int rc = row_grid(k, sm, g_warps<VPL>(), p.batch * p.n, nb)) return rc;
    k<<<nb, 32 * g_warps<VPL>(), sm, st>>>(p, o, lse);
    AFFMAE_LAUNCH_CHECK("gattn_fwd_row_kernel");
    return AFFMAE_OK;
}
template <int VPL>
static int row_fwd_launch(const GAttnP& p, int64_t width, __nv_bfloat16* o, float* lse, cudaStream_t st) {
    if (width <= 1) return row_fwd_launch2<VPL, 1>(p, o, lse, st);
    if constexpr (VPL >= 16) {  // not instantiated: 512-wide 8-slot rows take the thread kernel
        return fail(AFFMAE_EUNSUPPORTED, "gattn: internal routing");
    } else {
    auto k = gattn_fwd_reg_kernel<VPL, 8>;
    const size_t sm = size_t(p.heads) * p.hidden * sizeof(float4);
    unsigned nb = 0;
    if (int rc = row_grid(k, sm, 8, p.batch * p.n, nb)) return rc;
    k<<<nb, 256, sm, st>>>(p, o, lse);
    AFFMAE_LAUNCH_CHECK("gattn_fwd_reg_kernel");
    return AFFMAE_OK;
    }
}

template <int VPL, int MW, int UPL>
static int row_bwd_launch3(const GAttnP& p, cudaStream_t st, const __nv_bfloat16* g, __nv_bfloat16* q, float* dk,
                           float* dv, float* dbk, float* dbv, float* dw1, float* db1, float* dw2, float* db2,
                           float* dblank) {
    auto k = gattn_bwd_row_kernel<VPL, MW, UPL>;
    const size_t sm = row_smem<VPL, MW, true>(p);
    unsigned nb = 0;
    if (int rc = row_grid(k, sm, g_warps<VPL>(), p.batch * p.n, nb)) return rc;
    if (p.part && nb > unsigned(p.part_blocks)) nb = unsigned(p.part_blocks);
    k<<<nb, 32 * g_warps<VPL>(), sm, st>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    AFFMAE_LAUNCH_CHECK("gattn_bwd_row_kernel");
    if (p.part) {
        const int D = 32 * VPL, W = 2 * D + 4 * p.heads * p.hidden + 2 * p.heads;
        grow_reduce_kernel<<<(W + 255) / 256, 256, 0, st>>>(p.part, int(nb), W, D, p.heads, p.hidden, dbk, dbv, dw1,
                                                            db1, dw2, db2, dblank);
        AFFMAE_LAUNCH_CHECK("grow_reduce_kernel");
    }
    return AFFMAE_OK;
}
// (single-slot rows only: for the 8-slot rows the thread-per-(token, head) backward with the
// reverse-CSR dk / dv gather measured faster -- 1.48 vs 1.60 / 1.73 ms at 196608 x 8 rows)
template <int VPL>
static int row_bwd_launch(const GAttnP& p, int upl, cudaStream_t st, const __nv_bfloat16* g, __nv_bfloat16* q,
                          float* dk, float* dv, float* dbk, float* dbv, float* dw1, float* db1, float* dw2,
                          float* db2, float* dblank) {
    return upl <= 2 ? row_bwd_launch3<VPL, 1, 2>(p, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank)
                    : row_bwd_launch3<VPL, 1, 8>(p, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
}

int gattn_fwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx, const uint8_t* valid,
              int64_t batch, int64_t tokens, int64_t width, void* out, float* lse, void* stream, int64_t ldq,
              int64_t ldkv) {
    GAttnP p{};
    int rc = gattn_fill(p, a, in, idx, valid, batch, tokens, width);
    if (rc) return rc;
    if ((rc = gattn_strides(p, ldq, ldkv, 0, 0))) return rc;
    if (!out || !lse) return fail(AFFMAE_ECONFIG, "gattn: null output");
    if (batch == 0) return AFFMAE_OK;
    const size_t sm = size_t(a->heads) * a->bias_hidden * sizeof(float4);
    auto* o = static_cast<__nv_bfloat16*>(out);
    cudaStream_t st = as_stream(stream);
    switch (row_vpl(a, width)) {
        case 2: return row_fwd_launch<2>(p, width, o, lse, st);
        case 4: return row_fwd_launch<4>(p, width, o, lse, st);
        case 8: return row_fwd_launch<8>(p, width, o, lse, st);
        case 16:  // 512-wide 8-slot rows do not fit the register kernel (spills): thread kernel
            if (width <= 1) return row_fwd_launch<16>(p, width, o, lse, st);
            break;
        default: break;
    }
    const unsigned nb = gattn_blocks(batch * tokens, a->heads, 2048);
    const dim3 bt(32 * a->heads);
    if (a->head_dim == 16) gattn_fwd_kernel<16><<<nb, bt, sm, st>>>(p, o, lse);
    else if (a->head_dim == 32) gattn_fwd_kernel<32><<<nb, bt, sm, st>>>(p, o, lse);
    else gattn_fwd_kernel<64><<<nb, bt, sm, st>>>(p, o, lse);
    AFFMAE_LAUNCH_CHECK("gattn_fwd_kernel");
    return AFFMAE_OK;
}

template <int HD, bool G>
static void gattn_bwd_launch_g(int mw, unsigned nb, dim3 bt, size_t sm, cudaStream_t st, const GAttnP& p,
                               const __nv_bfloat16* g, __nv_bfloat16* q, float* dk, float* dv, float* dbk, float* dbv,
                               float* dw1, float* db1, float* dw2, float* db2, float* dblank) {
    if (mw <= 1) gattn_bwd_kernel<HD, 1, G><<<nb, bt, sm, st>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    else if (mw <= 8) gattn_bwd_kernel<HD, 8, G><<<nb, bt, sm, st>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    else if (mw <= 16) gattn_bwd_kernel<HD, 16, G><<<nb, bt, sm, st>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    else gattn_bwd_kernel<HD, 31, G><<<nb, bt, sm, st>>>(p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
}
template <int HD>
static void gattn_bwd_launch(int mw, unsigned nb, dim3 bt, size_t sm, cudaStream_t st, const GAttnP& p,
                             const __nv_bfloat16* g, __nv_bfloat16* q, float* dk, float* dv, float* dbk, float* dbv,
                             float* dw1, float* db1, float* dw2, float* db2, float* dblank) {
    if (p.dsw)
        gattn_bwd_launch_g<HD, true>(mw, nb, bt, sm, st, p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    else
        gattn_bwd_launch_g<HD, false>(mw, nb, bt, sm, st, p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
}

int gattn_bwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx, const uint8_t* valid,
              int64_t batch, int64_t tokens, int64_t width, const void* dout, void* dq, float* dk, float* dv,
              float* dbk, float* dbv, float* dw1, float* db1, float* dw2, float* db2, float* dblank, void* workspace,
              size_t ws_bytes, void* stream, int64_t ldq, int64_t ldkv, int64_t ldd) {
    GAttnP p{};
    int rc = gattn_fill(p, a, in, idx, valid, batch, tokens, width);
    if (rc) return rc;
    if ((rc = gattn_strides(p, ldq, ldkv, ldd, 0))) return rc;
    if (!dout || !dq || !dk || !dv || !dbk || !dbv || !dw1 || !db1 || !dw2 || !db2 || !dblank)
        return fail(AFFMAE_ECONFIG, "gattn bwd: null output");
    if (batch == 0) return AFFMAE_OK;
    const unsigned nb = gattn_blocks(batch * tokens, a->heads, 1024);
    const dim3 bt(32 * a->heads);
    // BiasNet units, then one 32 x 33 reduce-scatter tile per warp
    const size_t sm = size_t(a->heads) * a->bias_hidden * sizeof(float4) + size_t(a->heads) * 32 * 33 * sizeof(float);
    const auto* g = static_cast<const __nv_bfloat16*>(dout);
    auto* q = static_cast<__nv_bfloat16*>(dq);
    cudaStream_t st = as_stream(stream);
    const int mw = int(width);
    const bool gather = workspace != nullptr;
    int32_t *off = nullptr, *cur = nullptr, *ent = nullptr, *ent_key = nullptr;
    if (gather) {
        if (!gattn_gather_ok(a)) return fail(AFFMAE_EUNSUPPORTED, "gattn bwd: gather mode needs heads*head_dim in {32..512}");
        if (batch * tokens * width >= (int64_t(1) << 31)) return fail(AFFMAE_EUNSUPPORTED, "gattn bwd: too many entries");
        if (ws_bytes < gattn_bwd_workspace(a, batch, tokens, width)) return fail(AFFMAE_ECONFIG, "gattn bwd: workspace too small");
        const int64_t ents = batch * tokens * width;
        p.dsw = static_cast<float2*>(workspace);  // first: 8-byte aligned
        off = reinterpret_cast<int32_t*>(p.dsw + ents * a->heads);
        cur = off + batch * (tokens + 1);
        ent = cur + batch * tokens;
        ent_key = ent + ents;
        rev_csr_build(idx, valid, batch, tokens, tokens, mw, off, cur, ent, ent_key, st);
    }
    const int vpl = width <= 1 ? row_vpl(a, width) : 0;
    if (vpl) {
        const int upl = (a->bias_hidden + 32 / a->heads - 1) / (32 / a->heads);
        if (vpl == 2) rc = row_bwd_launch<2>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        else if (vpl == 4) rc = row_bwd_launch<4>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        else if (vpl == 8) rc = row_bwd_launch<8>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        else rc = row_bwd_launch<16>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        if (rc) return rc;
    } else {
        if (a->head_dim == 16) gattn_bwd_launch<16>(mw, nb, bt, sm, st, p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        else if (a->head_dim == 32) gattn_bwd_launch<32>(mw, nb, bt, sm, st, p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        else gattn_bwd_launch<64>(mw, nb, bt, sm, st, p, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
        AFFMAE_LAUNCH_CHECK("gattn_bwd_kernel");
    }
    if (gather) {
        const int64_t ents = batch * tokens * width;
        const unsigned gb = unsigned(std::max<int64_t>(1, std::min<int64_t>((ents + 255) / 256, 16 * kNumSMs)));
        const auto* qq = p.q;
        const int D = a->heads * a->head_dim;
#define AFFMAE_GG(D_)                                                                                           \
    case D_:                                                                                                    \
        gattn_kv_gather_kernel<D_><<<gb, 256, 0, st>>>(off, ent, ent_key, p.dsw, batch, tokens, mw, a->heads,   \
                                                       a->head_dim, qq, p.ldq, g, dk, dv);                      \
        break;
        switch (D) {
            AFFMAE_GG(32)
            AFFMAE_GG(64)
            AFFMAE_GG(128)
            AFFMAE_GG(256)
            AFFMAE_GG(512)
        }
#undef AFFMAE_GG
        AFFMAE_LAUNCH_CHECK("gattn_kv_gather_kernel");
    }
    return AFFMAE_OK;
}

int gattn_bwd_o2o(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx, const uint8_t* valid,
                  int64_t batch, int64_t tokens, const void* dout, void* dq, void* dk_bf16, void* dv_bf16, float* dbk,
                  float* dbv, float* dw1, float* db1, float* dw2, float* db2, float* dblank, void* workspace,
                  size_t ws_bytes, void* stream, int64_t ldq, int64_t ldkv, int64_t ldd, int64_t lddkv) {
    GAttnP p{};
    int rc = gattn_fill(p, a, in, idx, valid, batch, tokens, 1);
    if (rc) return rc;
    if ((rc = gattn_strides(p, ldq, ldkv, ldd, lddkv))) return rc;
    if (!dout || !dq || !dk_bf16 || !dv_bf16 || !dbk || !dbv || !dw1 || !db1 || !dw2 || !db2 || !dblank)
        return fail(AFFMAE_ECONFIG, "gattn bwd o2o: null output");
    const int vpl = row_vpl(a, 1);
    if (!vpl) return fail(AFFMAE_EUNSUPPORTED, "gattn bwd o2o: needs heads | 32 and heads*head_dim in {64..512}");
    if (batch == 0) return AFFMAE_OK;
    p.o2o = 1;
    if (workspace) {  // deterministic parameter gradients: per-block rows, reduced in block order
        const int W = 2 * a->heads * a->head_dim + 4 * a->heads * a->bias_hidden + 2 * a->heads;
        p.part = static_cast<float*>(workspace);
        p.part_blocks = int(std::min<size_t>(ws_bytes / (size_t(W) * 4), size_t(16 * device_sms())));
        if (p.part_blocks < 1) return fail(AFFMAE_ECONFIG, "gattn bwd o2o: workspace too small");
    }
    const int upl = (a->bias_hidden + 32 / a->heads - 1) / (32 / a->heads);
    const auto* g = static_cast<const __nv_bfloat16*>(dout);
    auto* q = static_cast<__nv_bfloat16*>(dq);
    auto* dk = static_cast<float*>(dk_bf16);
    auto* dv = static_cast<float*>(dv_bf16);
    cudaStream_t st = as_stream(stream);
    if (vpl == 2) return row_bwd_launch<2>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    if (vpl == 4) return row_bwd_launch<4>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    if (vpl == 8) return row_bwd_launch<8>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
    return row_bwd_launch<16>(p, upl, st, g, q, dk, dv, dbk, dbv, dw1, db1, dw2, db2, dblank);
}

}  // namespace affmae_b200
