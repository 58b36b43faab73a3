// Cluster attention kernels, forward and backward (replace nbhd_attn_streaming,
// nbhd_attn_backward and AttnOp: proj/src/attention.cpp:119-358,374-444).
//
// Work decomposition.  balanced_clusters puts the <= 16 members of cluster c
// at contiguous curve positions, and every member of c attends to the SAME
// key list: the concatenated members of nbr_cl[c][0..G) (own cluster first)
// plus one learned blank slot (proj/src/geometry.cpp:173-183,
// attention.cpp:152-156).  A cluster is therefore a small dense problem
//     S = Q_c (16 x d) . [K_nb ; blank_k]^T + bias,   O = softmax(S) . [V_nb ; blank_v]
// that maps onto one m16 tensor-core tile.
//
// Each kernel is persistent (grid = SMs x occupancy; blockIdx.y = head group
// of HPC heads, one warp per head) and walks (image, cluster) items:
//   1. token ids of the item were prefetched into registers one item ahead;
//   2. every gathered row (HPC*d bf16, 16-byte aligned) lands in padded shared
//      memory through ONE cp.async.bulk, completion counted in bytes on an
//      mbarrier (rows of the reference's NeighborIndex are gathered, no
//      per-row index arithmetic in the hot loop);
//   3. the relative-position bias + slot mask is evaluated ONCE per
//      (query, slot) pair for all HPC heads (one float4 lookup in the lattice
//      table, attn_common.cuh) straight into the mma accumulator fragment order,
//      so the score epilogue is one FFMA per element;
//   4. Q.K^T, P.V and the backward products run on bf16 mma.sync m16n8k16 with
//      fp32 accumulation; the whole <= 56-slot row stays in registers
//      (one-pass softmax == the reference's 16-slot online softmax).
//
// Backward, FA2-style and atomic-free for activations:
//   attn_bwd_dq_kernel   (per query cluster) recomputes P = exp(S - LSE),
//       dP = dO.V^T, D = rowsum(P o dP), dS = P (dP - D); writes dQ = dS.K/sqrt(d)
//       and D; blank grads; scatters dS into the bias-table gradient.
//   attn_bwd_dkdv_kernel (per key cluster c') stages the query clusters whose
//       neighbourhood holds c' (reverse CSR, ascending, up to KDEG per round)
//       and accumulates dK = dS^T.Q/sqrt(d), dV = P^T.dO in registers: each key
//       row is written once, in a fixed order (deterministic, no atomics).
#pragma once
#include <algorithm>

#include "attn_common.cuh"

namespace affmae_b200 {

struct AttnParams {
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    const __nv_bfloat16* bk;
    const __nv_bfloat16* bv;
    const float* coords;
    const int32_t* perm;
    const int32_t* keylist;  // [B*C][M+1]: key tokens in slot order (-1 pad), [M] = nk
    const int32_t* rev_off;  // [B][C+1]
    const int32_t* inq;      // [B][C*G][16]: query tokens of each reverse pair (-1 pad)
    const float* w1;
    const float* b1;
    const float* w2;
    const float* b2;
    const float* blank;
    const float* tab_g;  // [heads][kWg2]
    __nv_bfloat16* out;  // fwd output
    float* lse;          // fwd output / bwd input [B, N, heads]
    const __nv_bfloat16* dout;
    __nv_bfloat16* dq;
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    float* dsum;        // [B, N, heads]  D = rowsum(P o dP)
    float* dtab_g;      // [heads][kWg2]
    float* mlp_grad;    // [heads][4H+1]
    float* blank_grad;  // [heads][2d+1]  {dblank_k[d], dblank_v[d], dblank}
    ClusterShape cs;
    int batch;
    int heads;
    int hidden;
    float inv_patch;
    float scale;  // 1/sqrt(d)
};

template <int HPC> struct VecH;
template <> struct VecH<1> { using T = float; };
template <> struct VecH<2> { using T = float2; };
template <> struct VecH<4> { using T = float4; };
__device__ __forceinline__ float vget(float v, int) { return v; }
__device__ __forceinline__ float vget(float2 v, int i) { return i ? v.y : v.x; }
__device__ __forceinline__ float vget(float4 v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Shared lattice window of the bias table, heads interleaved, plus the
// tier-3 MLP parameters.
template <int HPC>
struct BiasTab {
    typename VecH<HPC>::T tab[kWs2];
    float4 units[HPC * kMaxHidden];
    float b2[HPC];
    float blank[HPC];
};

__device__ __forceinline__ void load_bias_tab(float* tab, float4* units, float* b2s, float* blanks,
                                              const AttnParams& p, int h0, int hpc) {
    for (int i = threadIdx.x; i < hpc * kWs2; i += blockDim.x) {
        int e = i / hpc, hh = i - e * hpc;
        int oy = e / kWs - kRs, ox = e % kWs - kRs;
        tab[i] = p.tab_g[size_t(h0 + hh) * kWg2 + (oy + kRg) * kWg + (ox + kRg)];
    }
    for (int i = threadIdx.x; i < hpc * p.hidden; i += blockDim.x) {
        int hh = i / p.hidden, u = i - hh * p.hidden, h = h0 + hh;
        units[hh * kMaxHidden + u] =
            make_float4(p.w1[h * 2 * p.hidden + u], p.w1[h * 2 * p.hidden + p.hidden + u],
                        p.b1[h * p.hidden + u], p.w2[h * p.hidden + u]);
    }
    for (int i = threadIdx.x; i < hpc; i += blockDim.x) {
        b2s[i] = p.b2[h0 + i];
        blanks[i] = p.blank[h0 + i];
    }
}

// Bias of pair (q, k) for all HPC heads.  Returns the window index (tier 1)
// or -1 (tiers 2/3 were evaluated).
template <int HPC>
__device__ __forceinline__ int pair_bias(const BiasTab<HPC>& bt, const AttnParams& p, int h0,
                                         const TokInfo& qi, const TokInfo& ki, float2 qxy,
                                         float2 kxy, float (&b)[HPC]) {
    int gi;
    int li = lut_index(qi, ki, gi);
    if (li >= 0) {
        typename VecH<HPC>::T v = bt.tab[li];
#pragma unroll
        for (int hh = 0; hh < HPC; ++hh) b[hh] = vget(v, hh);
    } else {
        const float ox = (kxy.x - qxy.x) * p.inv_patch, oy = (kxy.y - qxy.y) * p.inv_patch;
#pragma unroll
        for (int hh = 0; hh < HPC; ++hh)
            b[hh] = bias_tier23(p.tab_g + size_t(h0 + hh) * kWg2, gi, bt.units + hh * kMaxHidden,
                                p.hidden, bt.b2[hh], ox, oy);
    }
    return li;
}

__device__ __forceinline__ void item_coords(int item, int nc, int& img, int& c) {
    img = item / nc;
    c = item - img * nc;
}

// mma accumulator fragment <-> (row, col) of an m16 x (8*NT) tile
__device__ __forceinline__ void frag_pos(int f, int& row, int& col) {
    const int nt = f >> 7, ln = (f >> 2) & 31, e = f & 3;
    row = (ln >> 2) + ((e >> 1) << 3);
    col = nt * 8 + 2 * (ln & 3) + (e & 1);
}

// ===================================================== query-cluster side
template <int HD, int NT, int HPC, bool BWD>
struct QSmem {
    static constexpr int RW = HPC * HD + 8;
    static constexpr int NS = NT * 8;
    static constexpr int KVR = ((NT + 1) / 2) * 16;
    static constexpr int NF = NT * 128;
    static constexpr int MG = 4 * kMaxHidden + 1, BG = 2 * HD + 1;
    __nv_bfloat16 Q[16 * RW];
    __nv_bfloat16 K[KVR * RW];
    __nv_bfloat16 V[KVR * RW];
    __nv_bfloat16 dO[BWD ? 16 * RW : 8];
    float bias[HPC * NF];            // per head, fragment order; -inf = masked slot
    int32_t lidx[BWD ? NF : 4];      // table window index, -1 tier 2/3, -2 blank, -3 masked
    TokInfo qi[16];
    TokInfo ki[NS];
    float2 qxy[16];
    float2 kxy[NS];
    int32_t qtok[16];
    int32_t ktok[NS];
    float lse[BWD ? 16 * HPC : 4];
    float dtab[BWD ? HPC * kWs2 : 1];
    float mlpg[BWD ? HPC * MG : 1];
    float blankg[BWD ? HPC * BG : 1];
    float red[BWD ? HPC * 32 : 1];
    int32_t qlin[16];  // lattice cell iy*kWs + ix of each query
    int32_t klin[NS];  // ... and of each key slot
    int32_t meta[16];  // [0] nk; [1..12] lattice bbox / phase reductions; [13] fast
    const __nv_bfloat16* rowsrc[(BWD ? 32 : 16) + 2 * NS];  // gather source of every staged row
    BiasTab<HPC> bt;
};

// Item-level lattice check (meta[1..12]): every staged token shares one phase
// and every query/key offset lies inside the shared table window, so the
// window index of a pair is klin[slot] - qlin[row] + kWinC.
constexpr int kWinC = kRs * kWs + kRs;
__device__ __forceinline__ void lattice_meta_init(int32_t* meta) {
    for (int i = 1; i <= 12; ++i) meta[i] = (i & 1) ? INT32_MAX : INT32_MIN;  // odd: min, even: max
}
__device__ __forceinline__ void lattice_meta_add(int32_t* meta, const TokInfo& t, bool is_key) {
    int o = is_key ? 4 : 0;
    atomicMin(meta + 1 + o, t.ix);
    atomicMax(meta + 2 + o, t.ix);
    atomicMin(meta + 3 + o, t.iy);
    atomicMax(meta + 4 + o, t.iy);
    atomicMin(meta + 9, int(t.fx));
    atomicMax(meta + 10, int(t.fx));
    atomicMin(meta + 11, int(t.fy));
    atomicMax(meta + 12, int(t.fy));
}
__device__ __forceinline__ bool lattice_fast(const int32_t* meta) {
    return meta[9] == meta[10] && meta[11] == meta[12] && meta[6] - meta[1] <= kRs &&
           meta[2] - meta[5] <= kRs && meta[8] - meta[3] <= kRs && meta[4] - meta[7] <= kRs;
}

// Entry e of an item: e < 16 query token, 16 <= e < 16+NS key slot token,
// e == 16+NS the key count nk.  Held in registers one item ahead.
template <int NS, int NTHR>
struct TokPrefetch {
    static constexpr int E = 16 + NS + 1;
    static constexpr int PF = (E + NTHR - 1) / NTHR;
    int v[PF];
    __device__ __forceinline__ void load(const AttnParams& p, int item, int n_items) {
        if (item >= n_items) return;
        int img, c;
        item_coords(item, p.cs.c, img, c);
        const int M = p.cs.width;
        const int32_t* kl = p.keylist + int64_t(item) * (M + 1);
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            int e = threadIdx.x + j * NTHR, t = -1;
            if (e < 16) {
                if (e < p.cs.len(c)) t = p.perm[int64_t(img) * p.cs.n + p.cs.off(c) + e];
            } else if (e < 16 + NS) {
                if (e - 16 < M) t = kl[e - 16];
            } else if (e == 16 + NS) {
                t = kl[M];
            }
            v[j] = t;
        }
    }
};

template <typename SM>
__device__ __forceinline__ void zero_smem(SM& sm) {
    uint4* p = reinterpret_cast<uint4*>(&sm);
    for (int i = threadIdx.x; i < int(sizeof(SM) / 16); i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
}

// Installs the prefetched tokens of `item`, prefetches the next item, copies
// the rows (Q, dO, K, V, blanks) with cp.async (each thread owns one 16-byte
// column of every row: no per-chunk index math), stages lattice info / LSE
// and evaluates the bias fragments.  Ends with everything visible to the CTA.
template <int HD, int NT, int HPC, bool BWD>
__device__ __forceinline__ void stage_item(QSmem<HD, NT, HPC, BWD>& sm,
                                           const TokPrefetch<NT * 8, 32 * HPC>& pf,
                                           TokPrefetch<NT * 8, 32 * HPC>& pf_next,
                                           const AttnParams& p, int item, int next_item,
                                           int n_items, int h0) {
    using S = QSmem<HD, NT, HPC, BWD>;
    constexpr int NS = S::NS, RW = S::RW, NF = S::NF, NTHR = 32 * HPC;
    using PFT = TokPrefetch<NS, NTHR>;
    int img, c;
    item_coords(item, p.cs.c, img, c);
    const int64_t img_tok = int64_t(img) * p.cs.n;
    const int M = p.cs.width;
    const int tid = threadIdx.x;
    const int hd_all = p.heads * HD;

    __syncthreads();  // (A) previous item fully consumed
    float2 xy[PFT::PF];
    constexpr int QR = BWD ? 32 : 16;
#pragma unroll
    for (int j = 0; j < PFT::PF; ++j) {
        int e = tid + j * NTHR, t = pf.v[j];
        xy[j] = make_float2(0.f, 0.f);
        if (e < 16) {
            sm.qtok[e] = t;
            sm.rowsrc[e] = t >= 0 ? p.q + (img_tok + t) * hd_all + h0 * HD : nullptr;
            if (BWD) sm.rowsrc[16 + e] = t >= 0 ? p.dout + (img_tok + t) * hd_all + h0 * HD : nullptr;
        } else if (e < 16 + NS) {
            const int slot = e - 16;
            sm.ktok[slot] = t;
            sm.rowsrc[QR + slot] = t >= 0 ? p.k + (img_tok + t) * hd_all + h0 * HD
                                 : slot == M ? p.bk + h0 * HD : nullptr;
            sm.rowsrc[QR + NS + slot] = t >= 0 ? p.v + (img_tok + t) * hd_all + h0 * HD
                                      : slot == M ? p.bv + h0 * HD : nullptr;
        } else if (e == 16 + NS) {
            sm.meta[0] = t;
        }
        if (e < 16 + NS && t >= 0) xy[j] = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + t);
    }
    if (tid == 0) lattice_meta_init(sm.meta);
    float lse_v[HPC];
#pragma unroll
    for (int hh = 0; hh < HPC; ++hh) lse_v[hh] = INFINITY;
    if constexpr (BWD) {
        if (tid < 16 && pf.v[0] >= 0) {
            const float* lp = p.lse + (img_tok + pf.v[0]) * p.heads + h0;
#pragma unroll
            for (int hh = 0; hh < HPC; ++hh) lse_v[hh] = lp[hh];
        }
    }
    pf_next.load(p, next_item, n_items);
    __syncthreads();  // (B) tokens visible

    const int nk = sm.meta[0];
    {   // gather: one warp instruction moves 32 / CH whole rows (CH 16-byte chunks each)
        constexpr int CH = HPC * HD / 8, RPI = CH >= 32 ? 1 : 32 / CH, NW = NTHR / 32;
        constexpr int ROWS = QR + 2 * NS, GROUPS = (ROWS + RPI - 1) / RPI;
        const int wp = tid >> 5, ln = tid & 31, sub = ln / CH, ch = ln % CH;
        for (int gi = wp; gi < GROUPS; gi += NW) {
            const int r = gi * RPI + sub;
            if (sub < RPI && r < ROWS) {
                const __nv_bfloat16* src = sm.rowsrc[r];
                __nv_bfloat16* dst = r < 16 ? sm.Q + r * RW
                                   : r < QR ? sm.dO + (r - 16) * RW
                                   : r < QR + NS ? sm.K + (r - QR) * RW : sm.V + (r - QR - NS) * RW;
                if (src) cp_async16(dst + ch * 8, src + ch * 8);
                if (CH > 32)
                    for (int c2 = ch + 32; c2 < CH; c2 += 32)
                        if (src) cp_async16(dst + c2 * 8, src + c2 * 8);
            }
        }
        cp_async_commit();
    }
#pragma unroll
    for (int j = 0; j < PFT::PF; ++j) {
        int e = tid + j * NTHR;
        if (e < 16 + NS) {
            const TokInfo ti = make_tokinfo(xy[j], p.inv_patch);
            const int lin = ti.iy * kWs + ti.ix;
            const bool valid = e < 16 ? pf.v[j] >= 0 : (e - 16 < nk);
            if (e < 16) {
                sm.qxy[e] = xy[j];
                sm.qi[e] = ti;
                sm.qlin[e] = lin;
            } else {
                sm.kxy[e - 16] = xy[j];
                sm.ki[e - 16] = ti;
                sm.klin[e - 16] = lin;
            }
            if (valid) lattice_meta_add(sm.meta, ti, e >= 16);
        }
    }
    if constexpr (BWD) {
        if (tid < 16) {
#pragma unroll
            for (int hh = 0; hh < HPC; ++hh) sm.lse[tid * HPC + hh] = lse_v[hh];
        }
    }
    __syncthreads();  // (C) lattice info visible

    const bool fast = lattice_fast(sm.meta);
    for (int f = tid; f < NF; f += NTHR) {
        int row, slot;
        frag_pos(f, row, slot);
        float b[HPC];
        int li;
        if (slot < nk) {
            if (fast) {
                li = sm.klin[slot] - sm.qlin[row] + kWinC;
                const typename VecH<HPC>::T v = sm.bt.tab[li];
#pragma unroll
                for (int hh = 0; hh < HPC; ++hh) b[hh] = vget(v, hh);
            } else {
                li = pair_bias<HPC>(sm.bt, p, h0, sm.qi[row], sm.ki[slot], sm.qxy[row], sm.kxy[slot], b);
            }
        } else if (slot == M) {
            li = -2;
#pragma unroll
            for (int hh = 0; hh < HPC; ++hh) b[hh] = sm.bt.blank[hh];
        } else {
            li = -3;
#pragma unroll
            for (int hh = 0; hh < HPC; ++hh) b[hh] = -INFINITY;
        }
#pragma unroll
        for (int hh = 0; hh < HPC; ++hh) sm.bias[hh * NF + f] = b[hh];
        if constexpr (BWD) sm.lidx[f] = li;
    }
    if (tid == 0) sm.meta[13] = fast;
    cp_async_wait<0>();
    __syncthreads();  // (D) rows + bias fragments visible
}

// Scaled scores + bias + mask for one warp's head in accumulator layout:
// s[nt][e] <-> (row lane/4 + 8*(e>=2), slot nt*8 + 2*(lane%4) + (e&1)).
template <int HD, int NT, int HPC, bool BWD>
__device__ __forceinline__ void cluster_scores(const QSmem<HD, NT, HPC, BWD>& sm, float scale,
                                               int hh, float (&s)[NT][4]) {
    using S = QSmem<HD, NT, HPC, BWD>;
    constexpr int RW = S::RW, NF = S::NF;
    const int lane = threadIdx.x & 31;
    uint32_t qa[HD / 16][4];
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk)
        ldmatrix_x4(qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3],
                    sm.Q + (lane & 15) * RW + hh * HD + kk * 16 + (lane >> 4) * 8);
    const float4* bf = reinterpret_cast<const float4*>(sm.bias + hh * NF) + lane;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
        const __nv_bfloat16* kb = sm.K + (nt * 8 + (lane & 7)) * RW + hh * HD;
        if constexpr (HD >= 32) {
#pragma unroll
            for (int k2 = 0; k2 < HD / 32; ++k2) {
                uint32_t b[4];
                ldmatrix_x4(b[0], b[1], b[2], b[3], kb + k2 * 32 + (lane >> 3) * 8);
                mma_bf16_16816(s[nt], qa[2 * k2], b);
                mma_bf16_16816(s[nt], qa[2 * k2 + 1], b + 2);
            }
        } else {
            uint32_t b[2];
            ldmatrix_x2(b[0], b[1], kb + ((lane >> 3) & 1) * 8);
            mma_bf16_16816(s[nt], qa[0], b);
        }
        const float4 bb = bf[nt * 32];
        s[nt][0] = fmaf(s[nt][0], scale, bb.x);
        s[nt][1] = fmaf(s[nt][1], scale, bb.y);
        s[nt][2] = fmaf(s[nt][2], scale, bb.z);
        s[nt][3] = fmaf(s[nt][3], scale, bb.w);
    }
}

// ------------------------------------------------------------- forward
template <int HD, int NT, int HPC>
__global__ void __launch_bounds__(32 * HPC) attn_fwd_kernel(AttnParams p) {
    using SM = QSmem<HD, NT, HPC, false>;
    constexpr int RW = SM::RW, CH = HPC * HD / 8, NTHR = 32 * HPC;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    const int h0 = blockIdx.y * HPC;
    const int lane = threadIdx.x & 31, hh = threadIdx.x >> 5, h = h0 + hh;
    const int n_items = p.batch * p.cs.c;
    const int hd_all = p.heads * HD;
    zero_smem(sm);
    __syncthreads();
    load_bias_tab(reinterpret_cast<float*>(sm.bt.tab), sm.bt.units, sm.bt.b2, sm.bt.blank, p, h0, HPC);
    TokPrefetch<NT * 8, NTHR> pf[2];
    pf[0].load(p, blockIdx.x, n_items);
    int cur = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, cur ^= 1) {
        stage_item<HD, NT, HPC, false>(sm, pf[cur], pf[cur ^ 1], p, item, item + gridDim.x,
                                       n_items, h0);
        int img, c;
        item_coords(item, p.cs.c, img, c);
        float s[NT][4];
        cluster_scores<HD, NT, HPC, false>(sm, p.scale, hh, s);

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
        const float ms0 = m0 * kLog2e, ms1 = m1 * kLog2e;
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s[nt][0] = ex2_fast(fmaf(s[nt][0], kLog2e, -ms0));
            s[nt][1] = ex2_fast(fmaf(s[nt][1], kLog2e, -ms0));
            s[nt][2] = ex2_fast(fmaf(s[nt][2], kLog2e, -ms1));
            s[nt][3] = ex2_fast(fmaf(s[nt][3], kLog2e, -ms1));
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
#pragma unroll
        for (int ks = 0; ks < (NT + 1) / 2; ++ks) {
            uint32_t pa[4];
            pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
            pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
            if (2 * ks + 1 < NT) {
                pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
                pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
            } else {
                pa[2] = pa[3] = 0u;
            }
#pragma unroll
            for (int nd = 0; nd < HD / 8; nd += 2) {
                uint32_t b[4];
                ldmatrix_x4_trans(b[0], b[1], b[2], b[3],
                                  sm.V + (ks * 16 + (lane & 15)) * RW + hh * HD + nd * 8 +
                                      (lane >> 4) * 8);
                mma_bf16_16816(o[nd], pa, b);
                mma_bf16_16816(o[nd + 1], pa, b + 2);
            }
        }

        const float il0 = 1.f / l0, il1 = 1.f / l1;
        const int r0 = lane >> 2, c0 = 2 * (lane & 3);
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            *reinterpret_cast<uint32_t*>(sm.Q + r0 * RW + hh * HD + nd * 8 + c0) =
                pack_bf16(o[nd][0] * il0, o[nd][1] * il0);
            *reinterpret_cast<uint32_t*>(sm.Q + (r0 + 8) * RW + hh * HD + nd * 8 + c0) =
                pack_bf16(o[nd][2] * il1, o[nd][3] * il1);
        }
        const int qlen = p.cs.len(c);
        const int64_t img_tok = int64_t(img) * p.cs.n;
        if ((lane & 3) == 0) {
            if (r0 < qlen) p.lse[(img_tok + sm.qtok[r0]) * p.heads + h] = m0 + __logf(l0);
            if (r0 + 8 < qlen) p.lse[(img_tok + sm.qtok[r0 + 8]) * p.heads + h] = m1 + __logf(l1);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < qlen * CH; i += NTHR) {
            const int r = i / CH, ch = i % CH;
            *reinterpret_cast<uint4*>(p.out + (img_tok + sm.qtok[r]) * hd_all + h0 * HD + ch * 8) =
                *reinterpret_cast<const uint4*>(sm.Q + r * RW + ch * 8);
        }
    }
}

// ------------------------------------------------------- backward: dQ
template <int HD, int NT, int HPC>
__global__ void __launch_bounds__(32 * HPC) attn_bwd_dq_kernel(AttnParams p) {
    using SM = QSmem<HD, NT, HPC, true>;
    constexpr int RW = SM::RW, CH = HPC * HD / 8, NTHR = 32 * HPC, NF = SM::NF;
    constexpr int MG = SM::MG, BG = SM::BG;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    const int h0 = blockIdx.y * HPC;
    const int lane = threadIdx.x & 31, hh = threadIdx.x >> 5, h = h0 + hh;
    const int n_items = p.batch * p.cs.c;
    const int hd_all = p.heads * HD;
    const int M = p.cs.width;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    zero_smem(sm);
    __syncthreads();
    load_bias_tab(reinterpret_cast<float*>(sm.bt.tab), sm.bt.units, sm.bt.b2, sm.bt.blank, p, h0, HPC);
    float* mlpg = sm.mlpg + hh * MG;
    float* blankg = sm.blankg + hh * BG;
    float* red = sm.red + hh * 32;
    float* dtab_s = sm.dtab + hh * kWs2;
    float* dtab_g = p.dtab_g + size_t(h) * kWg2;
    TokPrefetch<NT * 8, NTHR> pf[2];
    pf[0].load(p, blockIdx.x, n_items);
    int cur = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, cur ^= 1) {
        stage_item<HD, NT, HPC, true>(sm, pf[cur], pf[cur ^ 1], p, item, item + gridDim.x,
                                      n_items, h0);
        int img, c;
        item_coords(item, p.cs.c, img, c);
        const int64_t img_tok = int64_t(img) * p.cs.n;
        const int qlen = p.cs.len(c);
        const int nk = sm.meta[0];
        const bool fast = sm.meta[13] != 0;

        float s[NT][4];
        cluster_scores<HD, NT, HPC, true>(sm, p.scale, hh, s);

        // dP = dO . V^T
        float dp[NT][4];
        {
            uint32_t oa[HD / 16][4];
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
                ldmatrix_x4(oa[kk][0], oa[kk][1], oa[kk][2], oa[kk][3],
                            sm.dO + (lane & 15) * RW + hh * HD + kk * 16 + (lane >> 4) * 8);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                dp[nt][0] = dp[nt][1] = dp[nt][2] = dp[nt][3] = 0.f;
                const __nv_bfloat16* vb = sm.V + (nt * 8 + (lane & 7)) * RW + hh * HD;
                if constexpr (HD >= 32) {
#pragma unroll
                    for (int k2 = 0; k2 < HD / 32; ++k2) {
                        uint32_t b[4];
                        ldmatrix_x4(b[0], b[1], b[2], b[3], vb + k2 * 32 + (lane >> 3) * 8);
                        mma_bf16_16816(dp[nt], oa[2 * k2], b);
                        mma_bf16_16816(dp[nt], oa[2 * k2 + 1], b + 2);
                    }
                } else {
                    uint32_t b[2];
                    ldmatrix_x2(b[0], b[1], vb + ((lane >> 3) & 1) * 8);
                    mma_bf16_16816(dp[nt], oa[0], b);
                }
            }
        }
        // P = exp(S - LSE);  D = rowsum(P o dP)
        const float ls0 = sm.lse[r0 * HPC + hh] * kLog2e;
        const float ls1 = sm.lse[(r0 + 8) * HPC + hh] * kLog2e;
        float D0 = 0.f, D1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s[nt][0] = ex2_fast(fmaf(s[nt][0], kLog2e, -ls0));
            s[nt][1] = ex2_fast(fmaf(s[nt][1], kLog2e, -ls0));
            s[nt][2] = ex2_fast(fmaf(s[nt][2], kLog2e, -ls1));
            s[nt][3] = ex2_fast(fmaf(s[nt][3], kLog2e, -ls1));
            D0 = fmaf(s[nt][0], dp[nt][0], fmaf(s[nt][1], dp[nt][1], D0));
            D1 = fmaf(s[nt][2], dp[nt][2], fmaf(s[nt][3], dp[nt][3], D1));
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            D0 += __shfl_xor_sync(0xffffffffu, D0, o);
            D1 += __shfl_xor_sync(0xffffffffu, D1, o);
        }
        if ((lane & 3) == 0) {
            if (r0 < qlen) p.dsum[(img_tok + sm.qtok[r0]) * p.heads + h] = D0;
            if (r0 + 8 < qlen) p.dsum[(img_tok + sm.qtok[r0 + 8]) * p.heads + h] = D1;
        }
        // dS = P (dP - D); blank column to scratch.  Bias-table gradient: on
        // lattice-fast items dS goes to smem (this head's bias slice, no longer
        // needed) and is scattered row by row below -- within one query row all
        // key offsets differ, so those shared-memory atomics never collide.
        const int4* lf = reinterpret_cast<const int4*>(sm.lidx) + lane;
        float4* dsf = reinterpret_cast<float4*>(sm.bias + hh * NF) + lane;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int4 l4 = lf[nt * 32];
            const int li[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool hi = e >= 2;
                const float pr = s[nt][e];
                const float ds = pr * (dp[nt][e] - (hi ? D1 : D0));
                const int row = hi ? r0 + 8 : r0;
                if (li[e] == -2) {
                    red[row] = ds;
                    red[16 + row] = pr;
                } else if (!fast && ds != 0.f) {
                    if (li[e] >= 0) {
                        atomicAdd(dtab_s + li[e], ds);
                    } else if (li[e] == -1) {
                        const int slot = nt * 8 + c0 + (e & 1);
                        int gi;
                        lut_index(sm.qi[row], sm.ki[slot], gi);
                        float2 kx = sm.kxy[slot], qx = sm.qxy[row];
                        bias_grad_tier23(dtab_g, gi, sm.bt.units + hh * kMaxHidden, p.hidden, ds,
                                         (kx.x - qx.x) * p.inv_patch, (kx.y - qx.y) * p.inv_patch, mlpg);
                    }
                }
                s[nt][e] = ds;
            }
            if (fast) dsf[nt * 32] = make_float4(s[nt][0], s[nt][1], s[nt][2], s[nt][3]);
        }
        if (fast) {
            __syncwarp();
            // Within one query row every key cell differs, so the offsets of a row
            // are distinct table entries: plain read-modify-write, no atomics.  A
            // duplicate key coordinate (two tokens on one cell) would alias two
            // lanes, so such items fall back to atomics.
            const int ka = lane < nk ? sm.klin[lane] : INT32_MIN + lane;
            const int kb = lane + 32 < nk ? sm.klin[lane + 32] : INT32_MIN + 32 + lane;
            const bool dup = __popc(__match_any_sync(0xffffffffu, ka)) > 1 ||
                             __popc(__match_any_sync(0xffffffffu, kb)) > 1;
            const bool dupw = __any_sync(0xffffffffu, dup);
            const float* dsr = sm.bias + hh * NF;
            for (int r = 0; r < qlen; ++r) {
                const int ql = kWinC - sm.qlin[r];
                const int fr = (((r & 7) << 2) << 2) + ((r >> 3) << 1);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int slot = lane + 32 * half;
                    if (slot < nk) {
                        const int f = ((slot >> 3) << 7) + fr + (((slot & 7) >> 1) << 2) + (slot & 1);
                        float* a = dtab_s + (half ? kb : ka) + ql;
                        const float v = dsr[f];
                        if (dupw) atomicAdd(a, v);
                        else *a += v;
                    }
                    __syncwarp();
                }
            }
        }
        __syncwarp();
        for (int d = lane; d < HD; d += 32) {
            float gk = 0.f, gv = 0.f;
#pragma unroll 4
            for (int r = 0; r < 16; ++r) {
                gk = fmaf(red[r], bf16_to_f32(*reinterpret_cast<const uint16_t*>(sm.Q + r * RW + hh * HD + d)), gk);
                gv = fmaf(red[16 + r], bf16_to_f32(*reinterpret_cast<const uint16_t*>(sm.dO + r * RW + hh * HD + d)), gv);
            }
            blankg[d] += gk * p.scale;
            blankg[HD + d] += gv;
        }
        if (lane == 0) {
            float sb = 0.f;
            for (int r = 0; r < 16; ++r) sb += red[r];
            blankg[2 * HD] += sb;
        }

        // dQ = dS . K / sqrt(d)
        float dqa[HD / 8][4];
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) dqa[nd][0] = dqa[nd][1] = dqa[nd][2] = dqa[nd][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < (NT + 1) / 2; ++ks) {
            uint32_t a[4];
            a[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
            a[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
            if (2 * ks + 1 < NT) {
                a[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
                a[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
            } else {
                a[2] = a[3] = 0u;
            }
#pragma unroll
            for (int nd = 0; nd < HD / 8; nd += 2) {
                uint32_t b[4];
                ldmatrix_x4_trans(b[0], b[1], b[2], b[3],
                                  sm.K + (ks * 16 + (lane & 15)) * RW + hh * HD + nd * 8 + (lane >> 4) * 8);
                mma_bf16_16816(dqa[nd], a, b);
                mma_bf16_16816(dqa[nd + 1], a, b + 2);
            }
        }
        __syncwarp();
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            *reinterpret_cast<uint32_t*>(sm.Q + r0 * RW + hh * HD + nd * 8 + c0) =
                pack_bf16(dqa[nd][0] * p.scale, dqa[nd][1] * p.scale);
            *reinterpret_cast<uint32_t*>(sm.Q + (r0 + 8) * RW + hh * HD + nd * 8 + c0) =
                pack_bf16(dqa[nd][2] * p.scale, dqa[nd][3] * p.scale);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < qlen * CH; i += NTHR) {
            const int r = i / CH, ch = i % CH;
            *reinterpret_cast<uint4*>(p.dq + (img_tok + sm.qtok[r]) * hd_all + h0 * HD + ch * 8) =
                *reinterpret_cast<const uint4*>(sm.Q + r * RW + ch * 8);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HPC * kWs2; i += NTHR) {
        float v = sm.dtab[i];
        if (v != 0.f) {
            int hq = i / kWs2, e = i - hq * kWs2;
            int oy = e / kWs - kRs, ox = e % kWs - kRs;
            atomicAdd(p.dtab_g + size_t(h0 + hq) * kWg2 + (oy + kRg) * kWg + (ox + kRg), v);
        }
    }
    for (int i = threadIdx.x; i < HPC * MG; i += NTHR) {
        int hq = i / MG, j = i - hq * MG;
        float v = sm.mlpg[i];
        if (j <= 4 * p.hidden && v != 0.f) atomicAdd(p.mlp_grad + (h0 + hq) * (4 * p.hidden + 1) + j, v);
    }
    for (int i = threadIdx.x; i < HPC * BG; i += NTHR) {
        int hq = i / BG, j = i - hq * BG;
        atomicAdd(p.blank_grad + (h0 + hq) * BG + j, sm.blankg[i]);
    }
}

// ===================================================== key-cluster side
constexpr int KDEG = 3;  // reverse pairs staged per round

template <int HD, int HPC>
struct KSmem {
    static constexpr int RW = HPC * HD + 8;
    static constexpr int NF = 256;  // 16 keys x 16 queries per pair
    __nv_bfloat16 K[16 * RW];
    __nv_bfloat16 V[16 * RW];
    __nv_bfloat16 Q[KDEG * 16 * RW];
    __nv_bfloat16 dO[KDEG * 16 * RW];
    float bias[KDEG * HPC * NF];  // [pair][head][fragment]
    TokInfo ki[16];
    TokInfo qi[KDEG * 16];
    float2 kxy[16];
    float2 qxy[KDEG * 16];
    int32_t ktok[16];
    int32_t qtok[KDEG * 16];
    float lse[KDEG * 16 * HPC];
    float dsum[KDEG * 16 * HPC];
    int32_t klin[16];
    int32_t qlin[KDEG * 16];
    int32_t meta[16];  // [14] rb, [15] re; [1..12] lattice reductions of the round
    uint64_t bar;
    BiasTab<HPC> bt;
};

template <int HD, int HPC>
__global__ void __launch_bounds__(32 * HPC) attn_bwd_dkdv_kernel(AttnParams p) {
    using S = KSmem<HD, HPC>;
    constexpr int RW = S::RW, CH = HPC * HD / 8, NTHR = 32 * HPC, NF = S::NF;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    S& sm = *reinterpret_cast<S*>(smem_raw);
    const int h0 = blockIdx.y * HPC;
    const int lane = threadIdx.x & 31, hh = threadIdx.x >> 5;
    const int tid = threadIdx.x;
    const ClusterShape& cs = p.cs;
    const int n_items = p.batch * cs.c;
    const int hd_all = p.heads * HD;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const int64_t pairs_per_img = int64_t(cs.c) * cs.g;
    zero_smem(sm);
    __syncthreads();
    load_bias_tab(reinterpret_cast<float*>(sm.bt.tab), sm.bt.units, sm.bt.b2, sm.bt.blank, p, h0, HPC);
    if (tid == 0) {
        mbar_init(&sm.bar, 1);
        fence_barrier_init();
    }
    uint32_t phase = 0;
    constexpr uint32_t ROWB = HPC * HD * 2;
    // item prefetch: key tokens (tid < 16), reverse range (tid 16, 17)
    auto item_pf = [&](int item) -> int {
        if (item >= n_items || tid >= 18) return -1;
        int img, ck;
        item_coords(item, cs.c, img, ck);
        if (tid < 16) return tid < cs.len(ck) ? p.perm[int64_t(img) * cs.n + cs.off(ck) + tid] : -1;
        return p.rev_off[int64_t(img) * (cs.c + 1) + ck + (tid - 16)];
    };
    int ipf = item_pf(blockIdx.x);
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int img, ck;
        item_coords(item, cs.c, img, ck);
        const int64_t img_tok = int64_t(img) * cs.n;
        const int klen = cs.len(ck);
        fence_proxy_async();
        __syncthreads();
        if (tid < 16) {
            sm.ktok[tid] = ipf;
            float2 kxy = make_float2(0.f, 0.f);
            if (ipf >= 0) kxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + ipf);
            const TokInfo ti = make_tokinfo(kxy, p.inv_patch);
            sm.kxy[tid] = kxy;
            sm.ki[tid] = ti;
            sm.klin[tid] = ti.iy * kWs + ti.ix;
        } else if (tid < 18) {
            sm.meta[14 + tid - 16] = ipf;
        }
        ipf = item_pf(item + gridDim.x);
        __syncthreads();
        const int rb = sm.meta[14], re = sm.meta[15];
        float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd)
#pragma unroll
            for (int e = 0; e < 4; ++e) dk[nd][e] = dv[nd][e] = 0.f;
        uint32_t ka[HD / 16][4], va[HD / 16][4];

        for (int rs = rb; rs < re; rs += KDEG) {
            const int np = min(KDEG, re - rs);
            const bool first = rs == rb;
            if (!first) {
                fence_proxy_async();
                __syncthreads();
            }
            // query tokens of this round, then their rows, coords, LSE and D
            for (int e = tid; e < KDEG * 16; e += NTHR)
                sm.qtok[e] = e < np * 16 ? p.inq[(int64_t(img) * pairs_per_img + rs) * 16 + e] : -1;
            if (tid == 0) lattice_meta_init(sm.meta);
            __syncthreads();
            if (tid == 0) {
                int nrows = 0;
                for (int i = 0; i < np * 16; ++i) nrows += sm.qtok[i] >= 0;
                mbar_arrive_expect_tx(&sm.bar, uint32_t(2 * nrows + (first ? 2 * klen : 0)) * ROWB);
            }
            for (int r = tid; r < np * 32 + (first ? 32 : 0); r += NTHR) {
                __nv_bfloat16* dst;
                const __nv_bfloat16* src = nullptr;
                if (r < np * 32) {
                    const bool isdo = r >= np * 16;
                    const int qr = isdo ? r - np * 16 : r, tok = sm.qtok[qr];
                    dst = (isdo ? sm.dO : sm.Q) + qr * RW;
                    if (tok >= 0) src = (isdo ? p.dout : p.q) + (img_tok + tok) * hd_all + h0 * HD;
                } else {
                    const int kr = r - np * 32;
                    const bool isv = kr >= 16;
                    const int tok = sm.ktok[kr & 15];
                    dst = (isv ? sm.V : sm.K) + (kr & 15) * RW;
                    if (tok >= 0) src = (isv ? p.v : p.k) + (img_tok + tok) * hd_all + h0 * HD;
                }
                if (src) bulk_g2s(dst, src, ROWB, &sm.bar);
            }
            for (int e = tid; e < np * 16; e += NTHR) {
                const int qt = sm.qtok[e];
                float2 qxy = make_float2(0.f, 0.f);
                float lv[HPC], dvv[HPC];
#pragma unroll
                for (int q = 0; q < HPC; ++q) { lv[q] = INFINITY; dvv[q] = 0.f; }
                if (qt >= 0) {
                    qxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + qt);
                    const float* lp = p.lse + (img_tok + qt) * p.heads + h0;
                    const float* dp_ = p.dsum + (img_tok + qt) * p.heads + h0;
#pragma unroll
                    for (int q = 0; q < HPC; ++q) { lv[q] = lp[q]; dvv[q] = dp_[q]; }
                }
                const TokInfo ti = make_tokinfo(qxy, p.inv_patch);
                sm.qxy[e] = qxy;
                sm.qi[e] = ti;
                sm.qlin[e] = ti.iy * kWs + ti.ix;
                if (qt >= 0) lattice_meta_add(sm.meta, ti, false);
#pragma unroll
                for (int q = 0; q < HPC; ++q) {
                    sm.lse[e * HPC + q] = lv[q];
                    sm.dsum[e * HPC + q] = dvv[q];
                }
            }
            for (int e = tid; e < klen; e += NTHR) lattice_meta_add(sm.meta, sm.ki[e], true);
            __syncthreads();
            // bias of (key row, query col) for every pair of the round, all heads
            const bool fast = lattice_fast(sm.meta);
            for (int f = tid; f < np * NF; f += NTHR) {
                const int pr = f >> 8, g = f & 255;
                int krow, qcol;
                frag_pos(g, krow, qcol);
                float b[HPC];
                if (fast) {
                    const typename VecH<HPC>::T v = sm.bt.tab[sm.klin[krow] - sm.qlin[pr * 16 + qcol] + kWinC];
#pragma unroll
                    for (int q = 0; q < HPC; ++q) b[q] = vget(v, q);
                } else {
                    pair_bias<HPC>(sm.bt, p, h0, sm.qi[pr * 16 + qcol], sm.ki[krow],
                                   sm.qxy[pr * 16 + qcol], sm.kxy[krow], b);
                }
#pragma unroll
                for (int q = 0; q < HPC; ++q) sm.bias[(pr * HPC + q) * NF + g] = b[q];
            }
            __syncthreads();
            mbar_wait(&sm.bar, phase);
            phase ^= 1;
            if (first) {
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    ldmatrix_x4(ka[kk][0], ka[kk][1], ka[kk][2], ka[kk][3],
                                sm.K + (lane & 15) * RW + hh * HD + kk * 16 + (lane >> 4) * 8);
                    ldmatrix_x4(va[kk][0], va[kk][1], va[kk][2], va[kk][3],
                                sm.V + (lane & 15) * RW + hh * HD + kk * 16 + (lane >> 4) * 8);
                }
            }
            for (int pr = 0; pr < np; ++pr) {
                const __nv_bfloat16* Qp = sm.Q + pr * 16 * RW;
                const __nv_bfloat16* Op = sm.dO + pr * 16 * RW;
                float sT[2][4], dpT[2][4];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) sT[nt][e] = dpT[nt][e] = 0.f;
                    const __nv_bfloat16* qb = Qp + (nt * 8 + (lane & 7)) * RW + hh * HD;
                    const __nv_bfloat16* ob = Op + (nt * 8 + (lane & 7)) * RW + hh * HD;
                    if constexpr (HD >= 32) {
#pragma unroll
                        for (int k2 = 0; k2 < HD / 32; ++k2) {
                            uint32_t b[4], bo[4];
                            ldmatrix_x4(b[0], b[1], b[2], b[3], qb + k2 * 32 + (lane >> 3) * 8);
                            ldmatrix_x4(bo[0], bo[1], bo[2], bo[3], ob + k2 * 32 + (lane >> 3) * 8);
                            mma_bf16_16816(sT[nt], ka[2 * k2], b);
                            mma_bf16_16816(sT[nt], ka[2 * k2 + 1], b + 2);
                            mma_bf16_16816(dpT[nt], va[2 * k2], bo);
                            mma_bf16_16816(dpT[nt], va[2 * k2 + 1], bo + 2);
                        }
                    } else {
                        uint32_t b[2], bo[2];
                        ldmatrix_x2(b[0], b[1], qb + ((lane >> 3) & 1) * 8);
                        ldmatrix_x2(bo[0], bo[1], ob + ((lane >> 3) & 1) * 8);
                        mma_bf16_16816(sT[nt], ka[0], b);
                        mma_bf16_16816(dpT[nt], va[0], bo);
                    }
                }
                const float4* bf = reinterpret_cast<const float4*>(sm.bias + (pr * HPC + hh) * NF) + lane;
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    const float4 bb = bf[nt * 32];
                    const float bv4[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int col = pr * 16 + nt * 8 + c0 + (e & 1);
                        const float pr_ = ex2_fast((fmaf(sT[nt][e], p.scale, bv4[e]) - sm.lse[col * HPC + hh]) * kLog2e);
                        sT[nt][e] = pr_;
                        dpT[nt][e] = pr_ * (dpT[nt][e] - sm.dsum[col * HPC + hh]);
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
                    ldmatrix_x4_trans(b[0], b[1], b[2], b[3], Op + (lane & 15) * RW + hh * HD + nd * 8 + (lane >> 4) * 8);
                    ldmatrix_x4_trans(bq[0], bq[1], bq[2], bq[3], Qp + (lane & 15) * RW + hh * HD + nd * 8 + (lane >> 4) * 8);
                    mma_bf16_16816(dv[nd], pa, b);
                    mma_bf16_16816(dv[nd + 1], pa, b + 2);
                    mma_bf16_16816(dk[nd], da, bq);
                    mma_bf16_16816(dk[nd + 1], da, bq + 2);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            *reinterpret_cast<uint32_t*>(sm.K + r0 * RW + hh * HD + nd * 8 + c0) =
                pack_bf16(dk[nd][0] * p.scale, dk[nd][1] * p.scale);
            *reinterpret_cast<uint32_t*>(sm.K + (r0 + 8) * RW + hh * HD + nd * 8 + c0) =
                pack_bf16(dk[nd][2] * p.scale, dk[nd][3] * p.scale);
            *reinterpret_cast<uint32_t*>(sm.V + r0 * RW + hh * HD + nd * 8 + c0) = pack_bf16(dv[nd][0], dv[nd][1]);
            *reinterpret_cast<uint32_t*>(sm.V + (r0 + 8) * RW + hh * HD + nd * 8 + c0) = pack_bf16(dv[nd][2], dv[nd][3]);
        }
        __syncthreads();
        for (int i = tid; i < 2 * klen * CH; i += NTHR) {
            const int r = i / CH, ch = i % CH;
            const bool isv = r >= klen;
            const int kr = isv ? r - klen : r;
            __nv_bfloat16* dst = (isv ? p.dv : p.dk) + (img_tok + sm.ktok[kr]) * hd_all + h0 * HD + ch * 8;
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>((isv ? sm.V : sm.K) + kr * RW + ch * 8);
        }
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
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (sms < 1) sms = kNumSMs;
    int per_group = std::max(1, occ * sms / hgroups);
    grid = dim3(unsigned(std::min(items, per_group)), unsigned(hgroups), 1);
    return AFFMAE_OK;
}

template <int HD, int NT, int HPC>
int launch_fwd(const AttnParams& p, cudaStream_t st) {
    auto kern = attn_fwd_kernel<HD, NT, HPC>;
    size_t smem = sizeof(QSmem<HD, NT, HPC, false>);
    dim3 grid;
    int rc = persistent_grid(kern, 32 * HPC, smem, p.batch * p.cs.c, p.heads / HPC, grid);
    if (rc) return rc;
    kern<<<grid, 32 * HPC, smem, st>>>(p);
    AFFMAE_LAUNCH_CHECK("attn_fwd_kernel");
    return AFFMAE_OK;
}

template <int HD, int NT, int HPC>
int launch_bwd(const AttnParams& p, cudaStream_t st) {
    {
        auto kern = attn_bwd_dq_kernel<HD, NT, HPC>;
        size_t smem = sizeof(QSmem<HD, NT, HPC, true>);
        dim3 grid;
        int rc = persistent_grid(kern, 32 * HPC, smem, p.batch * p.cs.c, p.heads / HPC, grid);
        if (rc) return rc;
        kern<<<grid, 32 * HPC, smem, st>>>(p);
        AFFMAE_LAUNCH_CHECK("attn_bwd_dq_kernel");
    }
    {
        auto kern = attn_bwd_dkdv_kernel<HD, HPC>;
        size_t smem = sizeof(KSmem<HD, HPC>);
        dim3 grid;
        int rc = persistent_grid(kern, 32 * HPC, smem, p.batch * p.cs.c, p.heads / HPC, grid);
        if (rc) return rc;
        kern<<<grid, 32 * HPC, smem, st>>>(p);
        AFFMAE_LAUNCH_CHECK("attn_bwd_dkdv_kernel");
    }
    return AFFMAE_OK;
}

#define AFFMAE_INSTANTIATE_ATTN(HD_, NT_, HPC_)                                   \
    template int launch_fwd<HD_, NT_, HPC_>(const AttnParams&, cudaStream_t); \
    template int launch_bwd<HD_, NT_, HPC_>(const AttnParams&, cudaStream_t);

}  // namespace affmae_b200
