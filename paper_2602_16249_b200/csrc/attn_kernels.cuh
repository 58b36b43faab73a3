// Cluster attention kernels, forward and backward (replace nbhd_attn_streaming,
// nbhd_attn_backward and AttnOp: proj/src/attention.cpp:119-358,374-444).
//
// Work decomposition.  balanced_clusters puts the <= 16 members of cluster c
// at contiguous curve positions, and every member of c attends to the SAME
// key list: the concatenated members of nbr_cl[c][0..G) (own cluster first)
// plus one learned blank slot (proj/src/geometry.cpp:173-183,
// attention.cpp:152-156).  A cluster is therefore a small dense problem
//     S = Q_c (16 x d) . [K_nb ; blank_k]^T + bias,   O = softmax(S) . [V_nb ; blank_v]
// on one m16 tensor-core tile (mma.sync m16n8k16 bf16, fp32 accumulate).
//
// Pipeline.  Every kernel is persistent (grid = SMs x resident CTAs; blockIdx.y
// = head group of HPC heads) and warp-specialised:
//   * one PRODUCER warp walks the CTA's items, copies the item's plan record
//     (token ids, lattice cells, flags; built once per call by the plan
//     kernels in attention.cu) into a ring stage and gathers every row the
//     item needs (HPC*d bf16 per token) with 16-byte cp.async, whose
//     completion the stage's `full` mbarrier tracks (cp.async.mbarrier.arrive);
//   * HPC CONSUMER warps (one per head) wait on `full`, run the tile maths
//     from shared memory, write their outputs and release the stage on
//     `empty`.
// With STAGES ring slots the gathers of the next item(s) overlap the maths of
// the current one; there is no CTA-wide barrier inside the item loop.
//
// Slot layout of a query-cluster item (KP = key slots rounded up to 16):
//   slots [0, nk) keys in reference order, [nk, KP) padding (masked),
//   slot KP the blank (K/V rows KP..KP+7 are static: blank row + zeros).
// The blank is one column of the score tile; its P.V contribution is a rank-1
// FFMA update (P_blank x blank_v), so V needs only KP rows in the forward.
//
// Relative-position bias (attn_common.cuh): on lattice-"fast" items (every
// token on one patch-lattice phase, every pair offset inside the shared
// window) the bias of (row, slot) is tab[kcell[slot] - qcell[row] + kWinC];
// all other items take an out-of-line exact path (window / global table /
// BiasNet MLP), so results are the same function for every input.
//
// Backward, FA2-style and atomic-free for activations:
//   attn_bwd_q_kernel  (per query cluster) recomputes P = exp(S - LSE),
//       dP = dO.V^T, D = rowsum(P o dP), dS = P (dP - D); writes dQ = dS.K/sqrt(d)
//       and D; blank grads (tensor-core rank-1 products); scatters dS into the
//       CTA's bias-table gradient window (row-major, conflict-free).
//   attn_bwd_kv_kernel (per key cluster c') walks the reverse-neighbour pairs
//       (query clusters whose neighbourhood holds c', ascending; up to KDEG per
//       ring stage) and accumulates dK = dS^T.Q/sqrt(d), dV = P^T.dO in
//       registers: every key row is written once, in a fixed order.
// Per-CTA parameter-gradient partials (bias-table window, blank, BiasNet MLP
// tier) go to a [CTA] buffer reduced in a fixed order afterwards: the
// backward is deterministic except for tier-2 (far-offset, same-phase) pairs.
#pragma once
#include <algorithm>

#include "attn_common.cuh"

namespace affmae_b200 {

// ------------------------------------------------------------ plan records
// Query-cluster item record, int32 words (built by attn_qrec_kernel).
template <int KP>
struct QRec {
    static constexpr int QTOK = 0, KTOK = 16, QCELL = 16 + KP, KCELL = 32 + KP, HDR = 32 + 2 * KP;
    static constexpr int WORDS = HDR + 8;  // multiple of 4 (16-byte rows)
};
enum { kHNk = 0, kHQlen = 1, kHFast = 2, kHDup0 = 3, kHDup1 = 4 };
// Key-cluster record: ktok[16] kcell[16] hdr{klen, rb, re}
struct KRec {
    static constexpr int KTOK = 0, KCELL = 16, HDR = 32, WORDS = 40;
};
// Reverse pair record (CSR order of rev_cl): qtok[16] qcell[16] hdr{qlen, fast}
struct PRec {
    static constexpr int QTOK = 0, QCELL = 16, HDR = 32, WORDS = 36;
};
constexpr int kWinC = kRs * kWs + kRs;  // window index of offset (0, 0)
constexpr int kMG = 4 * kMaxHidden + 1;  // tier-3 MLP grad accumulator per head

struct AttnParams {
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    const __nv_bfloat16* bk;
    const __nv_bfloat16* bv;
    const float* coords;
    const int32_t* qrec;     // [B*C][QRec::WORDS]
    const int32_t* krec;     // [B*C][KRec::WORDS]
    const int32_t* prec;     // [B][C*G][PRec::WORDS]
    const float* w1;
    const float* b1;
    const float* w2;
    const float* b2;
    const float* blank;
    const float* tab_g;  // [heads][kWg2] BiasNet at integer offsets
    __nv_bfloat16* out;  // fwd output
    float* lse;          // fwd output / bwd input [B, N, heads]
    const __nv_bfloat16* dout;
    __nv_bfloat16* dq;
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    float* dsum;     // [B, N, heads]  D = rowsum(P o dP)
    float* dtab_g;   // [heads][kWg2] tier-2 gradient (atomics)
    float* part;     // [CTAs][HPC][kPartW] per-CTA gradient partials
    ClusterShape cs;
    int batch;
    int heads;
    int hidden;
    float inv_patch;
    float scale;  // 1/sqrt(d)
};
// per-CTA, per-head partial: window dT [kWs2] | MLP grads [kMG] | blank {dbk[d], dbv[d], dblank}
__host__ __device__ constexpr int part_width(int hd) { return kWs2 + kMG + 2 * hd + 1; }

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ int4 ldg_nc4(const int32_t* p) {
    return __ldg(reinterpret_cast<const int4*>(p));
}
// Arrive on `bar` once every cp.async this thread issued so far has landed
// (pending count +1 now, -1 at completion: the phase cannot complete early).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Producer-warp row gather: `nrows` rows of ROWB bytes, row r from
// src(r) (global) to dst(r) (shared), as 16-byte cp.async -- each warp
// instruction moves 32 / (ROWB/16) whole rows.  (One cp.async.bulk per row
// is TMA-request-bound at these 128-256 B rows.)
template <int ROWB, typename SrcDst>
__device__ __forceinline__ void gather_rows(int nrows, int lane, SrcDst f) {
    constexpr int CPR = ROWB / 16, RPI = 32 / CPR;
    const int sub = lane / CPR, ch = lane - sub * CPR;
    for (int r = sub; r < nrows; r += RPI) {
        const __nv_bfloat16* src;
        __nv_bfloat16* dst;
        f(r, src, dst);
        cp_async16(dst + ch * 8, src + ch * 8);
    }
}

// Zero a shared-memory range (16-byte granules) with the whole CTA.
__device__ __forceinline__ void zero_shared(void* base, size_t bytes) {
    uint4* p = reinterpret_cast<uint4*>(base);
    for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
}

// Bias-table window of heads h0..h0+HPC into shared memory, pre-scaled by log2(e).
template <int HPC>
__device__ __forceinline__ void load_window(float* tab, const AttnParams& p, int h0) {
    for (int i = threadIdx.x; i < HPC * kWs2; i += blockDim.x) {
        const int hh = i / kWs2, e = i - hh * kWs2;
        const int oy = e / kWs - kRs, ox = e % kWs - kRs;
        tab[i] = p.tab_g[size_t(h0 + hh) * kWg2 + (oy + kRg) * kWg + (ox + kRg)] * kLog2e;
    }
}
// BiasNet MLP parameters (tier 3) of heads h0..h0+HPC.
template <int HPC>
__device__ __forceinline__ void load_units(float4* units, float* b2s, const AttnParams& p, int h0) {
    for (int i = threadIdx.x; i < HPC * p.hidden; i += blockDim.x) {
        const int hh = i / p.hidden, u = i - hh * p.hidden, h = h0 + hh;
        units[hh * kMaxHidden + u] =
            make_float4(p.w1[h * 2 * p.hidden + u], p.w1[h * 2 * p.hidden + p.hidden + u],
                        p.b1[h * p.hidden + u], p.w2[h * p.hidden + u]);
    }
    for (int i = threadIdx.x; i < HPC; i += blockDim.x) b2s[i] = p.b2[h0 + i];
}

// Exact bias (times log2 e) of one pair on a non-fast item: window, global
// table or the BiasNet MLP itself (tiers of attn_common.cuh).
static __device__ __noinline__ float slow_bias2(const AttnParams& p, const float* tab_s,
                                                const float4* units, float b2, int h,
                                                int64_t img_tok, int qt, int kt) {
    const float2 qxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + qt);
    const float2 kxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + kt);
    const TokInfo qi = make_tokinfo(qxy, p.inv_patch), ki = make_tokinfo(kxy, p.inv_patch);
    int gi;
    const int li = lut_index(qi, ki, gi);
    if (li >= 0) return tab_s[li];
    if (gi >= 0) return __ldg(p.tab_g + size_t(h) * kWg2 + gi) * kLog2e;
    return bias_mlp(units, p.hidden, b2, (kxy.x - qxy.x) * p.inv_patch, (kxy.y - qxy.y) * p.inv_patch) *
           kLog2e;
}
// Its gradient: += ds into the CTA window / the global table / the MLP partials.
static __device__ __noinline__ void slow_bias_grad(const AttnParams& p, float* dtab_s,
                                                   const float4* units, float* mlpg, int h,
                                                   int64_t img_tok, int qt, int kt, float ds) {
    const float2 qxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + qt);
    const float2 kxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + kt);
    const TokInfo qi = make_tokinfo(qxy, p.inv_patch), ki = make_tokinfo(kxy, p.inv_patch);
    int gi;
    const int li = lut_index(qi, ki, gi);
    if (li >= 0) atomicAdd(dtab_s + li, ds);
    else if (gi >= 0) atomicAdd(p.dtab_g + size_t(h) * kWg2 + gi, ds);
    else bias_mlp_grad(units, p.hidden, ds, (kxy.x - qxy.x) * p.inv_patch, (kxy.y - qxy.y) * p.inv_patch, mlpg);
}

// A-operand fragments of a 16-row tile (rows at stride RW, columns from `base`).
template <int HD, int RW>
__device__ __forceinline__ void load_a16(uint32_t (&a)[HD / 16][4], const __nv_bfloat16* base, int lane) {
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk)
        ldmatrix_x4(a[kk][0], a[kk][1], a[kk][2], a[kk][3], base + (lane & 15) * RW + kk * 16 + (lane >> 4) * 8);
}
// s[nt] = A(16 x HD) . B(rows nt*8 .. nt*8+7)^T for nt < NT.
template <int HD, int NT, int RW>
__device__ __forceinline__ void mma_abt(float (&s)[NT][4], const uint32_t (&a)[HD / 16][4],
                                        const __nv_bfloat16* b, int lane) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
        const __nv_bfloat16* kb = b + (nt * 8 + (lane & 7)) * RW;
        if constexpr (HD >= 32) {
#pragma unroll
            for (int k2 = 0; k2 < HD / 32; ++k2) {
                uint32_t bb[4];
                ldmatrix_x4(bb[0], bb[1], bb[2], bb[3], kb + k2 * 32 + (lane >> 3) * 8);
                mma_bf16_16816(s[nt], a[2 * k2], bb);
                mma_bf16_16816(s[nt], a[2 * k2 + 1], bb + 2);
            }
        } else {
            uint32_t bb[2];
            ldmatrix_x2(bb[0], bb[1], kb + ((lane >> 3) & 1) * 8);
            mma_bf16_16816(s[nt], a[0], bb);
        }
    }
}
// o += P(16 x 16*KS) . V(rows 0 .. 16*KS-1, HD); P in accumulator layout.
template <int HD, int KS, int NT, int RW>
__device__ __forceinline__ void mma_pv(float (&o)[HD / 8][4], const float (&pm)[NT][4],
                                       const __nv_bfloat16* v, int lane) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        uint32_t pa[4];
        pa[0] = pack_bf16(pm[2 * ks][0], pm[2 * ks][1]);
        pa[1] = pack_bf16(pm[2 * ks][2], pm[2 * ks][3]);
        pa[2] = pack_bf16(pm[2 * ks + 1][0], pm[2 * ks + 1][1]);
        pa[3] = pack_bf16(pm[2 * ks + 1][2], pm[2 * ks + 1][3]);
#pragma unroll
        for (int nd = 0; nd < HD / 8; nd += 2) {
            uint32_t b[4];
            ldmatrix_x4_trans(b[0], b[1], b[2], b[3], v + (ks * 16 + (lane & 15)) * RW + nd * 8 + (lane >> 4) * 8);
            mma_bf16_16816(o[nd], pa, b);
            mma_bf16_16816(o[nd + 1], pa, b + 2);
        }
    }
}
// Fragments (rows r0 / r0+8) -> bf16 rows in shared memory, scaled per row.
template <int HD, int RW>
__device__ __forceinline__ void frags_to_rows(__nv_bfloat16* sm, const float (&o)[HD / 8][4], float m0,
                                              float m1, int lane) {
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        *reinterpret_cast<uint32_t*>(sm + r0 * RW + nd * 8 + c0) = pack_bf16(o[nd][0] * m0, o[nd][1] * m0);
        *reinterpret_cast<uint32_t*>(sm + (r0 + 8) * RW + nd * 8 + c0) = pack_bf16(o[nd][2] * m1, o[nd][3] * m1);
    }
}
// Shared rows (this head's HD columns) -> global token rows, 16-byte stores.
template <int HD, int RW>
__device__ __forceinline__ void rows_to_global(__nv_bfloat16* g, int64_t img_tok, int hd_all, int hcol,
                                               const __nv_bfloat16* sm, const int32_t* tok, int nrows,
                                               int lane) {
    constexpr int CPR = HD / 8;
    for (int i = lane; i < nrows * CPR; i += 32) {
        const int r = i / CPR, ch = i - r * CPR;
        *reinterpret_cast<uint4*>(g + (img_tok + tok[r]) * hd_all + hcol + ch * 8) =
            *reinterpret_cast<const uint4*>(sm + r * RW + ch * 8);
    }
}

// Scaled scores + bias (log2 domain) + slot mask, accumulator layout:
// s[nt][e] <-> (row r0 + 8*(e>=2), slot nt*8 + c0 + (e&1)); tile KP/8 = blank.
template <int KP, int NT>
__device__ __forceinline__ void score_bias(float (&s)[NT][4], const int32_t* rec, const float* tab,
                                           float scale2, float blank2, int nk, bool fast, int lane,
                                           const AttnParams& p, const float4* units, float b2,
                                           int h, int64_t img_tok) {
    using R = QRec<KP>;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    if (fast) {
        const int q0 = kWinC - rec[R::QCELL + r0], q1 = kWinC - rec[R::QCELL + r0 + 8];
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) {
            const int2 kc = *reinterpret_cast<const int2*>(rec + R::KCELL + nt * 8 + c0);
            s[nt][0] = fmaf(s[nt][0], scale2, tab[kc.x + q0]);
            s[nt][1] = fmaf(s[nt][1], scale2, tab[kc.y + q0]);
            s[nt][2] = fmaf(s[nt][2], scale2, tab[kc.x + q1]);
            s[nt][3] = fmaf(s[nt][3], scale2, tab[kc.y + q1]);
        }
    } else {
        const int qt0 = rec[R::QTOK + r0], qt1 = rec[R::QTOK + r0 + 8];
        const int qa = qt0 >= 0 ? qt0 : rec[R::QTOK], qb = qt1 >= 0 ? qt1 : rec[R::QTOK];
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int slot = nt * 8 + c0 + (e & 1);
                const int kt = slot < nk ? rec[R::KTOK + slot] : rec[R::KTOK];
                s[nt][e] = fmaf(s[nt][e], scale2,
                                slow_bias2(p, tab, units, b2, h, img_tok, e >= 2 ? qb : qa, kt));
            }
        }
    }
    if (nk < KP) {
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) {
            const int sl = nt * 8 + c0;
            if (sl >= nk) s[nt][0] = s[nt][2] = -INFINITY;
            if (sl + 1 >= nk) s[nt][1] = s[nt][3] = -INFINITY;
        }
    }
    const bool bl = c0 == 0;
    s[NT - 1][0] = bl ? fmaf(s[NT - 1][0], scale2, blank2) : -INFINITY;
    s[NT - 1][2] = bl ? fmaf(s[NT - 1][2], scale2, blank2) : -INFINITY;
    s[NT - 1][1] = s[NT - 1][3] = -INFINITY;
}

// ======================================================= forward
template <int HD, int KP, int HPC>
struct FwdCfg {
    static constexpr int RW = HPC * HD + 8;          // padded row (bf16 elements)
    static constexpr uint32_t ROWB = HPC * HD * 2;  // bytes per gathered row
    static constexpr int NT = KP / 8 + 1;
    static constexpr int QW = QRec<KP>::WORDS;
    static constexpr int STAGES = 2;
    struct alignas(16) Stage {
        __nv_bfloat16 Q[16 * RW];
        __nv_bfloat16 K[(KP + 8) * RW];
        __nv_bfloat16 V[KP * RW];
        int32_t rec[QW];
        uint64_t full, empty;
        uint64_t pad_;
    };
    struct alignas(16) Smem {
        Stage st[STAGES];
        float tab[HPC * kWs2];
        float4 units[HPC * kMaxHidden];
        float b2[HPC];
    };
};

template <int HD, int KP, int HPC>
__global__ void __launch_bounds__(32 * (HPC + 1)) attn_fwd_kernel(AttnParams p) {
    using C = FwdCfg<HD, KP, HPC>;
    using R = QRec<KP>;
    constexpr int RW = C::RW, NT = C::NT, S = C::STAGES;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
    const int h0 = blockIdx.y * HPC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = p.batch * p.cs.c;
    const int hd_all = p.heads * HD;

    zero_shared(sm.st, sizeof(sm.st));
    __syncthreads();
    for (int i = threadIdx.x; i < S * HPC * HD; i += blockDim.x) {
        const int s = i / (HPC * HD), j = i - s * (HPC * HD);
        sm.st[s].K[KP * RW + j] = p.bk[h0 * HD + j];  // blank key row; rows KP+1.. stay 0
    }
    load_window<HPC>(sm.tab, p, h0);
    load_units<HPC>(sm.units, sm.b2, p, h0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&sm.st[s].full, 32);
            mbar_init(&sm.st[s].empty, HPC);
        }
        fence_barrier_init();
    }
    fence_proxy_async();
    __syncthreads();

    if (warp == HPC) {  // ------------------------------------------ producer
        int it = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
            auto& st = sm.st[it % S];
            if (it >= S) mbar_wait(&st.empty, ((it / S) & 1) ^ 1);
            const int32_t* g = p.qrec + size_t(item) * C::QW;
            for (int w = lane * 4; w < C::QW; w += 128) *reinterpret_cast<int4*>(st.rec + w) = ldg_nc4(g + w);
            const int nk = __ldg(g + R::HDR + kHNk), qlen = __ldg(g + R::HDR + kHQlen);
            const __nv_bfloat16* qb = p.q + int64_t(item / p.cs.c) * p.cs.n * hd_all + h0 * HD;
            const __nv_bfloat16* kb = p.k + (qb - p.q);
            const __nv_bfloat16* vb = p.v + (qb - p.q);
            __syncwarp();
            const int32_t* rec = st.rec;
            gather_rows<C::ROWB>(qlen + 2 * nk, lane, [&](int r, const __nv_bfloat16*& src, __nv_bfloat16*& dst) {
                if (r < qlen) {
                    src = qb + int64_t(rec[R::QTOK + r]) * hd_all;
                    dst = st.Q + r * RW;
                } else {
                    const bool isv = r >= qlen + nk;
                    const int sl = r - qlen - (isv ? nk : 0);
                    src = (isv ? vb : kb) + int64_t(rec[R::KTOK + sl]) * hd_all;
                    dst = (isv ? st.V : st.K) + sl * RW;
                }
            });
            cp_async_mbar_arrive(&st.full);
            mbar_arrive(&st.full);
        }
        return;
    }

    // --------------------------------------------------------- consumers
    const int hh = warp, h = h0 + hh;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const float scale2 = p.scale * kLog2e, blank2 = p.blank[h] * kLog2e;
    const float* tab = sm.tab + hh * kWs2;
    float bvr[HD / 8][2];
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        bvr[nd][0] = __bfloat162float(p.bv[h * HD + nd * 8 + c0]);
        bvr[nd][1] = __bfloat162float(p.bv[h * HD + nd * 8 + c0 + 1]);
    }
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        auto& st = sm.st[it % S];
        mbar_wait(&st.full, (it / S) & 1);
        const int32_t* rec = st.rec;
        const int nk = rec[R::HDR + kHNk], qlen = rec[R::HDR + kHQlen];
        const bool fast = rec[R::HDR + kHFast] != 0;
        const int64_t img_tok = int64_t(item / p.cs.c) * p.cs.n;

        uint32_t qa[HD / 16][4];
        load_a16<HD, RW>(qa, st.Q + hh * HD, lane);
        float s[NT][4];
        mma_abt<HD, NT, RW>(s, qa, st.K + hh * HD, lane);
        score_bias<KP, NT>(s, rec, tab, scale2, blank2, nk, fast, lane, p, sm.units + hh * kMaxHidden,
                           sm.b2[hh], h, img_tok);

        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            m0 = fmaxf(m0, fmaxf(s[nt][0], s[nt][1]));
            m1 = fmaxf(m1, fmaxf(s[nt][2], s[nt][3]));
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
            m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
        }
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s[nt][0] = ex2_fast(s[nt][0] - m0);
            s[nt][1] = ex2_fast(s[nt][1] - m0);
            s[nt][2] = ex2_fast(s[nt][2] - m1);
            s[nt][3] = ex2_fast(s[nt][3] - m1);
            l0 += s[nt][0] + s[nt][1];
            l1 += s[nt][2] + s[nt][3];
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        float o[HD / 8][4];
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
        mma_pv<HD, KP / 16, NT, RW>(o, s, st.V + hh * HD, lane);
        // blank slot: rank-1 update P_blank x blank_v
        const float pb0 = __shfl_sync(0xffffffffu, s[NT - 1][0], lane & ~3);
        const float pb1 = __shfl_sync(0xffffffffu, s[NT - 1][2], lane & ~3);
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            o[nd][0] = fmaf(pb0, bvr[nd][0], o[nd][0]);
            o[nd][1] = fmaf(pb0, bvr[nd][1], o[nd][1]);
            o[nd][2] = fmaf(pb1, bvr[nd][0], o[nd][2]);
            o[nd][3] = fmaf(pb1, bvr[nd][1], o[nd][3]);
        }
        frags_to_rows<HD, RW>(st.Q + hh * HD, o, 1.f / l0, 1.f / l1, lane);
        if ((lane & 3) == 0) {
            if (r0 < qlen) p.lse[(img_tok + rec[R::QTOK + r0]) * p.heads + h] = (m0 + __log2f(l0)) * kLn2;
            if (r0 + 8 < qlen) p.lse[(img_tok + rec[R::QTOK + r0 + 8]) * p.heads + h] = (m1 + __log2f(l1)) * kLn2;
        }
        __syncwarp();
        rows_to_global<HD, RW>(p.out, img_tok, hd_all, h * HD, st.Q + hh * HD, rec + R::QTOK, qlen, lane);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&st.empty);
    }
}

// ======================================================= backward, query side
template <int HD, int KP, int HPC>
struct BwdQCfg {
    static constexpr int RW = HPC * HD + 8;
    static constexpr uint32_t ROWB = HPC * HD * 2;
    static constexpr int NT = KP / 8 + 1;
    static constexpr int QW = QRec<KP>::WORDS;
    static constexpr int STAGES = 2;
    struct alignas(16) Stage {
        __nv_bfloat16 Q[16 * RW];
        __nv_bfloat16 dO[16 * RW];
        __nv_bfloat16 K[(KP + 8) * RW];
        __nv_bfloat16 V[(KP + 8) * RW];
        int32_t rec[QW];
        float lse[16 * HPC];
        uint64_t full, empty;
    };
    struct alignas(16) Smem {
        Stage st[STAGES];
        float tab[HPC * kWs2];
        float dtab[HPC * kWs2];
        float scr[HPC * 8 * KP];  // dS rows of one half tile, per head
        float4 units[HPC * kMaxHidden];
        float mlpg[HPC * kMG];
        float b2[HPC];
    };
};

template <int HD, int KP, int HPC>
__global__ void __launch_bounds__(32 * (HPC + 1)) attn_bwd_q_kernel(AttnParams p) {
    using C = BwdQCfg<HD, KP, HPC>;
    using R = QRec<KP>;
    constexpr int RW = C::RW, NT = C::NT, S = C::STAGES;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
    const int h0 = blockIdx.y * HPC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = p.batch * p.cs.c;
    const int hd_all = p.heads * HD;

    zero_shared(&sm, sizeof(sm));
    __syncthreads();
    for (int i = threadIdx.x; i < S * HPC * HD; i += blockDim.x) {
        const int s = i / (HPC * HD), j = i - s * (HPC * HD);
        sm.st[s].K[KP * RW + j] = p.bk[h0 * HD + j];
        sm.st[s].V[KP * RW + j] = p.bv[h0 * HD + j];
    }
    load_window<HPC>(sm.tab, p, h0);
    load_units<HPC>(sm.units, sm.b2, p, h0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&sm.st[s].full, 32);
            mbar_init(&sm.st[s].empty, HPC);
        }
        fence_barrier_init();
    }
    fence_proxy_async();
    __syncthreads();

    if (warp == HPC) {  // ------------------------------------------ producer
        int it = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
            auto& st = sm.st[it % S];
            if (it >= S) mbar_wait(&st.empty, ((it / S) & 1) ^ 1);
            const int32_t* g = p.qrec + size_t(item) * C::QW;
            for (int w = lane * 4; w < C::QW; w += 128) *reinterpret_cast<int4*>(st.rec + w) = ldg_nc4(g + w);
            const int nk = __ldg(g + R::HDR + kHNk), qlen = __ldg(g + R::HDR + kHQlen);
            const int64_t img_tok = int64_t(item / p.cs.c) * p.cs.n;
            const int qt = lane < qlen ? __ldg(g + R::QTOK + lane) : -1;
            if (lane < 16) {
#pragma unroll
                for (int hq = 0; hq < HPC; ++hq)
                    st.lse[lane * HPC + hq] = qt >= 0 ? __ldg(p.lse + (img_tok + qt) * p.heads + h0 + hq) : INFINITY;
            }
            __syncwarp();
            const int32_t* rec = st.rec;
            const int64_t ib = int64_t(item / p.cs.c) * p.cs.n * hd_all + h0 * HD;
            gather_rows<C::ROWB>(2 * qlen + 2 * nk, lane, [&](int r, const __nv_bfloat16*& src, __nv_bfloat16*& dst) {
                if (r < 2 * qlen) {
                    const bool iso = r >= qlen;
                    const int qr = r - (iso ? qlen : 0);
                    src = (iso ? p.dout : p.q) + ib + int64_t(rec[R::QTOK + qr]) * hd_all;
                    dst = (iso ? st.dO : st.Q) + qr * RW;
                } else {
                    const bool isv = r >= 2 * qlen + nk;
                    const int sl = r - 2 * qlen - (isv ? nk : 0);
                    src = (isv ? p.v : p.k) + ib + int64_t(rec[R::KTOK + sl]) * hd_all;
                    dst = (isv ? st.V : st.K) + sl * RW;
                }
            });
            cp_async_mbar_arrive(&st.full);
            mbar_arrive(&st.full);
        }
        return;
    }

    // --------------------------------------------------------- consumers
    const int hh = warp, h = h0 + hh;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const float scale2 = p.scale * kLog2e, blank2 = p.blank[h] * kLog2e;
    const float* tab = sm.tab + hh * kWs2;
    float* dtab = sm.dtab + hh * kWs2;
    float* scr = sm.scr + hh * 8 * KP;
    float* mlpg = sm.mlpg + hh * kMG;
    const float4* units = sm.units + hh * kMaxHidden;
    float bkr[HD / 8][2];
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        bkr[nd][0] = __bfloat162float(p.bk[h * HD + nd * 8 + c0]);
        bkr[nd][1] = __bfloat162float(p.bk[h * HD + nd * 8 + c0 + 1]);
    }
    float gbk[HD / 8][2], gbv[HD / 8][2];  // blank grads, row 0 of a rank-1 mma (lanes 0..3)
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) gbk[nd][0] = gbk[nd][1] = gbv[nd][0] = gbv[nd][1] = 0.f;
    float gblank = 0.f;

    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        auto& st = sm.st[it % S];
        mbar_wait(&st.full, (it / S) & 1);
        const int32_t* rec = st.rec;
        const int nk = rec[R::HDR + kHNk], qlen = rec[R::HDR + kHQlen];
        const bool fast = rec[R::HDR + kHFast] != 0;
        const int64_t img_tok = int64_t(item / p.cs.c) * p.cs.n;

        uint32_t qa[HD / 16][4], oa[HD / 16][4];
        load_a16<HD, RW>(qa, st.Q + hh * HD, lane);
        load_a16<HD, RW>(oa, st.dO + hh * HD, lane);
        float s[NT][4], dp[NT][4];
        mma_abt<HD, NT, RW>(s, qa, st.K + hh * HD, lane);
        mma_abt<HD, NT, RW>(dp, oa, st.V + hh * HD, lane);
        score_bias<KP, NT>(s, rec, tab, scale2, blank2, nk, fast, lane, p, units, sm.b2[hh], h, img_tok);

        // P = exp(S - LSE);  D = rowsum(P o dP)
        const float ls0 = st.lse[r0 * HPC + hh] * kLog2e, ls1 = st.lse[(r0 + 8) * HPC + hh] * kLog2e;
        float D0 = 0.f, D1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s[nt][0] = ex2_fast(s[nt][0] - ls0);
            s[nt][1] = ex2_fast(s[nt][1] - ls0);
            s[nt][2] = ex2_fast(s[nt][2] - ls1);
            s[nt][3] = ex2_fast(s[nt][3] - ls1);
            D0 = fmaf(s[nt][0], dp[nt][0], fmaf(s[nt][1], dp[nt][1], D0));
            D1 = fmaf(s[nt][2], dp[nt][2], fmaf(s[nt][3], dp[nt][3], D1));
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            D0 += __shfl_xor_sync(0xffffffffu, D0, o);
            D1 += __shfl_xor_sync(0xffffffffu, D1, o);
        }
        if ((lane & 3) == 0) {
            if (r0 < qlen) p.dsum[(img_tok + rec[R::QTOK + r0]) * p.heads + h] = D0;
            if (r0 + 8 < qlen) p.dsum[(img_tok + rec[R::QTOK + r0 + 8]) * p.heads + h] = D1;
        }
        // dS = P (dP - D), in place of P; keep the blank column's P
        const float pbl0 = s[NT - 1][0], pbl1 = s[NT - 1][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s[nt][0] *= dp[nt][0] - D0;
            s[nt][1] *= dp[nt][1] - D0;
            s[nt][2] *= dp[nt][2] - D1;
            s[nt][3] *= dp[nt][3] - D1;
        }
        // ---- blank grads: dblank += sum dS_b; dbk += dS_b^T Q; dbv += P_b^T dO (rank-1 mma)
        {
            const float dsb0 = s[NT - 1][0], dsb1 = s[NT - 1][2];
            if (c0 == 0) gblank += dsb0 + dsb1;
            const int src = 8 * (lane & 3);
            const float x0 = __shfl_sync(0xffffffffu, dsb0, src), x1 = __shfl_sync(0xffffffffu, dsb0, src + 4);
            const float x2 = __shfl_sync(0xffffffffu, dsb1, src), x3 = __shfl_sync(0xffffffffu, dsb1, src + 4);
            const float y0 = __shfl_sync(0xffffffffu, pbl0, src), y1 = __shfl_sync(0xffffffffu, pbl0, src + 4);
            const float y2 = __shfl_sync(0xffffffffu, pbl1, src), y3 = __shfl_sync(0xffffffffu, pbl1, src + 4);
            const bool row0 = lane < 4;
            const uint32_t ax[4] = {row0 ? pack_bf16(x0, x1) : 0u, 0u, row0 ? pack_bf16(x2, x3) : 0u, 0u};
            const uint32_t ay[4] = {row0 ? pack_bf16(y0, y1) : 0u, 0u, row0 ? pack_bf16(y2, y3) : 0u, 0u};
#pragma unroll
            for (int nd = 0; nd < HD / 8; nd += 2) {
                uint32_t b[4], bo[4];
                ldmatrix_x4_trans(b[0], b[1], b[2], b[3], st.Q + (lane & 15) * RW + hh * HD + nd * 8 + (lane >> 4) * 8);
                ldmatrix_x4_trans(bo[0], bo[1], bo[2], bo[3], st.dO + (lane & 15) * RW + hh * HD + nd * 8 + (lane >> 4) * 8);
                float t0[4] = {0.f, 0.f, 0.f, 0.f}, t1[4] = {0.f, 0.f, 0.f, 0.f};
                float u0[4] = {0.f, 0.f, 0.f, 0.f}, u1[4] = {0.f, 0.f, 0.f, 0.f};
                mma_bf16_16816(t0, ax, b);
                mma_bf16_16816(t1, ax, b + 2);
                mma_bf16_16816(u0, ay, bo);
                mma_bf16_16816(u1, ay, bo + 2);
                gbk[nd][0] += t0[0];
                gbk[nd][1] += t0[1];
                gbk[nd + 1][0] += t1[0];
                gbk[nd + 1][1] += t1[1];
                gbv[nd][0] += u0[0];
                gbv[nd][1] += u0[1];
                gbv[nd + 1][0] += u1[0];
                gbv[nd + 1][1] += u1[1];
            }
        }
        // ---- dQ = dS . K / sqrt(d)  (+ blank rank-1 dS_b x blank_k)
        float dqa[HD / 8][4];
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) dqa[nd][0] = dqa[nd][1] = dqa[nd][2] = dqa[nd][3] = 0.f;
        mma_pv<HD, KP / 16, NT, RW>(dqa, s, st.K + hh * HD, lane);
        {
            const float b0 = __shfl_sync(0xffffffffu, s[NT - 1][0], lane & ~3);
            const float b1 = __shfl_sync(0xffffffffu, s[NT - 1][2], lane & ~3);
#pragma unroll
            for (int nd = 0; nd < HD / 8; ++nd) {
                dqa[nd][0] = fmaf(b0, bkr[nd][0], dqa[nd][0]);
                dqa[nd][1] = fmaf(b0, bkr[nd][1], dqa[nd][1]);
                dqa[nd][2] = fmaf(b1, bkr[nd][0], dqa[nd][2]);
                dqa[nd][3] = fmaf(b1, bkr[nd][1], dqa[nd][3]);
            }
        }
        // ---- bias-table gradient
        if (fast) {
            // Rows of one query hold pairwise-distinct key cells, so a row-major
            // pass writes distinct window entries per instruction: plain RMW
            // (duplicate key coordinates -> the rec flags force atomics).
            const bool dup0 = rec[R::HDR + kHDup0] != 0, dup1 = rec[R::HDR + kHDup1] != 0;
            const int ka = lane < nk ? rec[R::KCELL + lane] + kWinC : 0;
            const int kb = lane + 32 < nk ? rec[R::KCELL + lane + 32] + kWinC : 0;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
#pragma unroll
                for (int nt = 0; nt < KP / 8; ++nt)
                    *reinterpret_cast<float2*>(scr + r0 * KP + nt * 8 + c0) =
                        make_float2(s[nt][2 * half], s[nt][2 * half + 1]);
                __syncwarp();
                const int rows = min(8, qlen - 8 * half);
                for (int rr = 0; rr < rows; ++rr) {
                    const int qc = rec[R::QCELL + 8 * half + rr];
                    if (lane < nk) {
                        float* a = dtab + ka - qc;
                        const float v = scr[rr * KP + lane];
                        if (dup0) atomicAdd(a, v);
                        else *a += v;
                    }
                    __syncwarp();
                    if (KP > 32 && lane + 32 < nk) {
                        float* a = dtab + kb - qc;
                        const float v = scr[rr * KP + lane + 32];
                        if (dup1) atomicAdd(a, v);
                        else *a += v;
                    }
                    __syncwarp();
                }
            }
        } else {
#pragma unroll
            for (int nt = 0; nt < KP / 8; ++nt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int row = r0 + ((e >> 1) << 3), slot = nt * 8 + c0 + (e & 1);
                    if (row < qlen && slot < nk && s[nt][e] != 0.f)
                        slow_bias_grad(p, dtab, units, mlpg, h, img_tok, rec[R::QTOK + row],
                                       rec[R::KTOK + slot], s[nt][e]);
                }
            }
        }
        // ---- write dQ (this head's columns) through the stage's Q rows
        __syncwarp();
        frags_to_rows<HD, RW>(st.Q + hh * HD, dqa, p.scale, p.scale, lane);
        __syncwarp();
        rows_to_global<HD, RW>(p.dq, img_tok, hd_all, h * HD, st.Q + hh * HD, rec + R::QTOK, qlen, lane);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&st.empty);
    }

    // ---- per-CTA partials (reduced in a fixed order by attn_part_reduce_kernel)
    __syncwarp();
    float* part = p.part + (size_t(blockIdx.y) * gridDim.x + blockIdx.x) * HPC * part_width(HD) +
                  size_t(hh) * part_width(HD);
    for (int i = lane; i < kWs2; i += 32) part[i] = dtab[i];
    for (int i = lane; i < kMG; i += 32) part[kWs2 + i] = mlpg[i];
    float* pb = part + kWs2 + kMG;
    gblank += __shfl_xor_sync(0xffffffffu, gblank, 4);
    gblank += __shfl_xor_sync(0xffffffffu, gblank, 8);
    gblank += __shfl_xor_sync(0xffffffffu, gblank, 16);
    if (lane < 4) {
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            pb[nd * 8 + 2 * lane] = gbk[nd][0] * p.scale;
            pb[nd * 8 + 2 * lane + 1] = gbk[nd][1] * p.scale;
            pb[HD + nd * 8 + 2 * lane] = gbv[nd][0];
            pb[HD + nd * 8 + 2 * lane + 1] = gbv[nd][1];
        }
    }
    if (lane == 0) pb[2 * HD] = gblank;
}

// ======================================================= backward, key side
constexpr int KDEG = 3;  // reverse pairs per ring stage

template <int HD, int HPC>
struct BwdKCfg {
    static constexpr int RW = HPC * HD + 8;
    static constexpr uint32_t ROWB = HPC * HD * 2;
    static constexpr int STAGES = 2;
    static constexpr int LQ = KDEG * 16;
    struct alignas(16) Stage {
        __nv_bfloat16 K[16 * RW];
        __nv_bfloat16 V[16 * RW];
        __nv_bfloat16 Q[LQ * RW];
        __nv_bfloat16 dO[LQ * RW];
        float lse[HPC * LQ];  // [head][pair*16 + query], log2 domain
        float dsum[HPC * LQ];
        int32_t krec[KRec::WORDS];
        int32_t prec[KDEG * PRec::WORDS];
        int32_t hdr[4];  // item (-1: end), np, first, last
        uint64_t full, empty;
    };
    struct alignas(16) Smem {
        Stage st[STAGES];
        float tab[HPC * kWs2];
        float4 units[HPC * kMaxHidden];
        float b2[HPC];
    };
};

template <int HD, int HPC>
__global__ void __launch_bounds__(32 * (HPC + 1)) attn_bwd_kv_kernel(AttnParams p) {
    using C = BwdKCfg<HD, HPC>;
    constexpr int RW = C::RW, S = C::STAGES, LQ = C::LQ;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
    const int h0 = blockIdx.y * HPC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = p.batch * p.cs.c;
    const int hd_all = p.heads * HD;
    const int pairs_per_img = p.cs.c * p.cs.g;

    zero_shared(sm.st, sizeof(sm.st));
    __syncthreads();
    load_window<HPC>(sm.tab, p, h0);
    load_units<HPC>(sm.units, sm.b2, p, h0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&sm.st[s].full, 32);
            mbar_init(&sm.st[s].empty, HPC);
        }
        fence_barrier_init();
    }
    fence_proxy_async();
    __syncthreads();

    if (warp == HPC) {  // ------------------------------------------ producer
        int rr = 0;
        auto acquire = [&](int r) -> typename C::Stage& {
            auto& st = sm.st[r % S];
            if (r >= S) mbar_wait(&st.empty, ((r / S) & 1) ^ 1);
            return st;
        };
        for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
            const int img = item / p.cs.c;
            const int64_t img_tok = int64_t(img) * p.cs.n;
            const int32_t* kg = p.krec + size_t(item) * KRec::WORDS;
            const int klen = __ldg(kg + KRec::HDR), rb = __ldg(kg + KRec::HDR + 1), re = __ldg(kg + KRec::HDR + 2);
            for (int rs = rb; rs < re; rs += KDEG, ++rr) {
                auto& st = acquire(rr);
                const int np = min(KDEG, re - rs);
                const bool first = rs == rb;
                for (int w = lane * 4; w < KRec::WORDS; w += 128)
                    *reinterpret_cast<int4*>(st.krec + w) = ldg_nc4(kg + w);
                const int32_t* pg = p.prec + (size_t(img) * pairs_per_img + rs) * PRec::WORDS;
                for (int w = lane * 4; w < np * PRec::WORDS; w += 128)
                    *reinterpret_cast<int4*>(st.prec + w) = ldg_nc4(pg + w);
                if (lane == 0) {
                    st.hdr[0] = item;
                    st.hdr[1] = np;
                    st.hdr[2] = first;
                    st.hdr[3] = rs + KDEG >= re;
                }
                // LSE / D of the round's queries: lane -> (pair e/16, query e%16)
#pragma unroll
                for (int j = 0; j < (LQ + 31) / 32; ++j) {
                    const int e = lane + 32 * j, pr = e >> 4, qi = e & 15;
                    if (e < LQ) {
                        const int qt = pr < np ? __ldg(pg + pr * PRec::WORDS + PRec::QTOK + qi) : -1;
#pragma unroll
                        for (int hq = 0; hq < HPC; ++hq) {
                            st.lse[hq * LQ + e] =
                                qt >= 0 ? __ldg(p.lse + (img_tok + qt) * p.heads + h0 + hq) * kLog2e : INFINITY;
                            st.dsum[hq * LQ + e] = qt >= 0 ? __ldg(p.dsum + (img_tok + qt) * p.heads + h0 + hq) : 0.f;
                        }
                    }
                }
                __syncwarp();
                // rows: [K 16 | V 16] on the item's first round, then per pair [Q 16 | dO 16]
                const int kv = first ? 32 : 0;
                const int64_t ib = img_tok * hd_all + h0 * HD;
                constexpr int CPR = C::ROWB / 16, RPI = 32 / CPR;
                const int sub = lane / CPR, ch = lane - sub * CPR;
                for (int r = sub; r < kv + np * 32; r += RPI) {
                    int tok;
                    const __nv_bfloat16* src;
                    __nv_bfloat16* dst;
                    if (r < kv) {
                        const int kr = r & 15;
                        tok = st.krec[KRec::KTOK + kr];
                        src = r < 16 ? p.k : p.v;
                        dst = (r < 16 ? st.K : st.V) + kr * RW;
                    } else {
                        const int x = r - kv, pr = x >> 5, qi = x & 15;
                        tok = st.prec[pr * PRec::WORDS + PRec::QTOK + qi];
                        src = (x & 16) ? p.dout : p.q;
                        dst = ((x & 16) ? st.dO : st.Q) + (pr * 16 + qi) * RW;
                    }
                    if (tok >= 0) cp_async16(dst + ch * 8, src + ib + int64_t(tok) * hd_all + ch * 8);
                }
                cp_async_mbar_arrive(&st.full);
                mbar_arrive(&st.full);
            }
        }
        // end marker
        auto& st = acquire(rr);
        if (lane == 0) st.hdr[0] = -1;
        __syncwarp();
        mbar_arrive(&st.full);
        return;
    }

    // --------------------------------------------------------- consumers
    const int hh = warp, h = h0 + hh;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const float scale2 = p.scale * kLog2e;
    const float* tab = sm.tab + hh * kWs2;
    const float4* units = sm.units + hh * kMaxHidden;
    uint32_t ka[HD / 16][4], va[HD / 16][4];
    float dk[HD / 8][4], dv[HD / 8][4];
    int kq0 = 0, kq1 = 0, klen = 0, kt0 = 0, kt1 = 0;
    for (int rr = 0;; ++rr) {
        auto& st = sm.st[rr % S];
        mbar_wait(&st.full, (rr / S) & 1);
        const int item = st.hdr[0];
        if (item < 0) break;
        const int np = st.hdr[1];
        const bool first = st.hdr[2] != 0, last = st.hdr[3] != 0;
        const int64_t img_tok = int64_t(item / p.cs.c) * p.cs.n;
        if (first) {
            load_a16<HD, RW>(ka, st.K + hh * HD, lane);
            load_a16<HD, RW>(va, st.V + hh * HD, lane);
#pragma unroll
            for (int nd = 0; nd < HD / 8; ++nd)
#pragma unroll
                for (int e = 0; e < 4; ++e) dk[nd][e] = dv[nd][e] = 0.f;
            klen = st.krec[KRec::HDR];
            kq0 = st.krec[KRec::KCELL + r0] + kWinC;
            kq1 = st.krec[KRec::KCELL + r0 + 8] + kWinC;
            kt0 = st.krec[KRec::KTOK + (r0 < klen ? r0 : 0)];
            kt1 = st.krec[KRec::KTOK + (r0 + 8 < klen ? r0 + 8 : 0)];
        }
        for (int pr = 0; pr < np; ++pr) {
            const __nv_bfloat16* Qp = st.Q + pr * 16 * RW + hh * HD;
            const __nv_bfloat16* Op = st.dO + pr * 16 * RW + hh * HD;
            const int32_t* prc = st.prec + pr * PRec::WORDS;
            float sT[2][4], dpT[2][4];
            mma_abt<HD, 2, RW>(sT, ka, Qp, lane);
            mma_abt<HD, 2, RW>(dpT, va, Op, lane);
            const bool fast = prc[PRec::HDR + 1] != 0;
            const float* lsp = st.lse + hh * LQ + pr * 16;
            const float* dsp = st.dsum + hh * LQ + pr * 16;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int qc = nt * 8 + c0;
                float b[4];
                if (fast) {
                    const int2 qcl = *reinterpret_cast<const int2*>(prc + PRec::QCELL + qc);
                    b[0] = tab[kq0 - qcl.x];
                    b[1] = tab[kq0 - qcl.y];
                    b[2] = tab[kq1 - qcl.x];
                    b[3] = tab[kq1 - qcl.y];
                } else {
                    const int qlen = prc[PRec::HDR];
                    const int qa = prc[PRec::QTOK + (qc < qlen ? qc : 0)];
                    const int qb = prc[PRec::QTOK + (qc + 1 < qlen ? qc + 1 : 0)];
                    b[0] = slow_bias2(p, tab, units, sm.b2[hh], h, img_tok, qa, kt0);
                    b[1] = slow_bias2(p, tab, units, sm.b2[hh], h, img_tok, qb, kt0);
                    b[2] = slow_bias2(p, tab, units, sm.b2[hh], h, img_tok, qa, kt1);
                    b[3] = slow_bias2(p, tab, units, sm.b2[hh], h, img_tok, qb, kt1);
                }
                const float2 l2 = *reinterpret_cast<const float2*>(lsp + qc);
                const float2 d2 = *reinterpret_cast<const float2*>(dsp + qc);
                const float lv[4] = {l2.x, l2.y, l2.x, l2.y}, dvv[4] = {d2.x, d2.y, d2.x, d2.y};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float pr_ = ex2_fast(fmaf(sT[nt][e], scale2, b[e]) - lv[e]);
                    sT[nt][e] = pr_;
                    dpT[nt][e] = pr_ * (dpT[nt][e] - dvv[e]);
                }
            }
            uint32_t pa[4], da[4];
            pa[0] = pack_bf16(sT[0][0], sT[0][1]);
            pa[1] = pack_bf16(sT[0][2], sT[0][3]);
            pa[2] = pack_bf16(sT[1][0], sT[1][1]);
            pa[3] = pack_bf16(sT[1][2], sT[1][3]);
            da[0] = pack_bf16(dpT[0][0], dpT[0][1]);
            da[1] = pack_bf16(dpT[0][2], dpT[0][3]);
            da[2] = pack_bf16(dpT[1][0], dpT[1][1]);
            da[3] = pack_bf16(dpT[1][2], dpT[1][3]);
#pragma unroll
            for (int nd = 0; nd < HD / 8; nd += 2) {
                uint32_t b[4], bq[4];
                ldmatrix_x4_trans(b[0], b[1], b[2], b[3], Op + (lane & 15) * RW + nd * 8 + (lane >> 4) * 8);
                ldmatrix_x4_trans(bq[0], bq[1], bq[2], bq[3], Qp + (lane & 15) * RW + nd * 8 + (lane >> 4) * 8);
                mma_bf16_16816(dv[nd], pa, b);
                mma_bf16_16816(dv[nd + 1], pa, b + 2);
                mma_bf16_16816(dk[nd], da, bq);
                mma_bf16_16816(dk[nd + 1], da, bq + 2);
            }
        }
        if (last) {
            __syncwarp();
            frags_to_rows<HD, RW>(st.K + hh * HD, dk, p.scale, p.scale, lane);
            frags_to_rows<HD, RW>(st.V + hh * HD, dv, 1.f, 1.f, lane);
            __syncwarp();
            rows_to_global<HD, RW>(p.dk, img_tok, hd_all, h * HD, st.K + hh * HD, st.krec + KRec::KTOK, klen, lane);
            rows_to_global<HD, RW>(p.dv, img_tok, hd_all, h * HD, st.V + hh * HD, st.krec + KRec::KTOK, klen, lane);
            fence_proxy_async();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&st.empty);
    }
}

// ------------------------------------------------------------ launchers
template <typename K>
inline int persistent_grid(K kern, int threads, size_t smem, int items, int hgroups, dim3& grid) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
    }
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (e != cudaSuccess) return cuda_status(e, "occupancy");
    if (occ < 1) return fail(AFFMAE_EUNSUPPORTED, "attention: kernel does not fit on an SM");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = kNumSMs;
    const int per_group = std::max(1, std::min(occ * sms / hgroups, kMaxCtasPerGroup));
    grid = dim3(unsigned(std::min(items, per_group)), unsigned(hgroups), 1);
    return AFFMAE_OK;
}

template <int HD, int KP, int HPC>
int launch_fwd(const AttnParams& p, cudaStream_t st) {
    auto kern = attn_fwd_kernel<HD, KP, HPC>;
    const size_t smem = sizeof(typename FwdCfg<HD, KP, HPC>::Smem);
    dim3 grid;
    int rc = persistent_grid(kern, 32 * (HPC + 1), smem, p.batch * p.cs.c, p.heads / HPC, grid);
    if (rc) return rc;
    kern<<<grid, 32 * (HPC + 1), smem, st>>>(p);
    AFFMAE_LAUNCH_CHECK("attn_fwd_kernel");
    return AFFMAE_OK;
}

// Launches the query-side kernel; `grid_x` returns its CTA count per head group.
template <int HD, int KP, int HPC>
int launch_bwd_q(const AttnParams& p, cudaStream_t st, int& grid_x) {
    auto kern = attn_bwd_q_kernel<HD, KP, HPC>;
    const size_t smem = sizeof(typename BwdQCfg<HD, KP, HPC>::Smem);
    dim3 grid;
    int rc = persistent_grid(kern, 32 * (HPC + 1), smem, p.batch * p.cs.c, p.heads / HPC, grid);
    if (rc) return rc;
    kern<<<grid, 32 * (HPC + 1), smem, st>>>(p);
    AFFMAE_LAUNCH_CHECK("attn_bwd_q_kernel");
    grid_x = int(grid.x);
    return AFFMAE_OK;
}

template <int HD, int HPC>
int launch_bwd_kv(const AttnParams& p, cudaStream_t st) {
    auto kern = attn_bwd_kv_kernel<HD, HPC>;
    const size_t smem = sizeof(typename BwdKCfg<HD, HPC>::Smem);
    dim3 grid;
    int rc = persistent_grid(kern, 32 * (HPC + 1), smem, p.batch * p.cs.c, p.heads / HPC, grid);
    if (rc) return rc;
    kern<<<grid, 32 * (HPC + 1), smem, st>>>(p);
    AFFMAE_LAUNCH_CHECK("attn_bwd_kv_kernel");
    return AFFMAE_OK;
}

#define AFFMAE_INSTANTIATE_ATTN_QK(HD_, KP_, HPC_)                                   \
    template int launch_fwd<HD_, KP_, HPC_>(const AttnParams&, cudaStream_t); \
    template int launch_bwd_q<HD_, KP_, HPC_>(const AttnParams&, cudaStream_t, int&);
#define AFFMAE_INSTANTIATE_ATTN_KV(HD_, HPC_) \
    template int launch_bwd_kv<HD_, HPC_>(const AttnParams&, cudaStream_t);

}  // namespace affmae_b200
