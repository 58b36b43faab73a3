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
// Execution model: warp-autonomous.  A CTA is ONE warp that owns ONE head
// (blockIdx.y) and walks the items blockIdx.x, +gridDim.x, ... (persistent
// grid, ~SMs x resident warps).  The warp gathers only its head's d-column
// slice of every row (HD*2 bytes: 8 rows per 16-byte cp.async instruction at
// d = 32) into padded shared rows (ldmatrix conflict-free), so warps never
// wait on each other -- the heads of a token row are independent slices.
// Software pipeline, per warp, with cp.async groups:
//     plan record of item i+2 -> record ring (3)      (issued at iteration i)
//     rows of item i+1        -> row ring (2)         (tokens from record i+1)
//     compute item i                                  (rows landed: wait_group 2)
// so the gathers of the next item overlap the maths of the current one and
// the record latency is hidden two items deep.
//
// Slot layout of a query-cluster item (KP = key slots rounded up to 16):
//   slots [0, nk) keys in reference order, [nk, KP) padding (masked),
//   slot KP the blank: a static 8-row tile (blank row + zeros) forms the last
//   n-tile of the score product; its P.V / dS.K contributions are rank-1
//   FFMA updates, so the row ring holds only KP key/value rows.
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
//       warp's bias-table gradient window (row-major, conflict-free).
//   attn_bwd_kv_kernel (per key cluster c') walks the reverse-neighbour pairs
//       (query clusters whose neighbourhood holds c', ascending), one pair per
//       pipeline round, and accumulates dK = dS^T.Q/sqrt(d), dV = P^T.dO in
//       registers: every key row is written once, in a fixed order.
// Per-warp parameter-gradient partials (bias-table window, blank, BiasNet MLP
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
    static constexpr int WORDS = HDR + 8;  // multiple of 4 (16-byte copies)
};
enum { kHNk = 0, kHQlen = 1, kHFast = 2, kHDup0 = 3, kHDup1 = 4, kHImgTok = 5, kHItem = 6 };  // img_tok = image * N
// Key-cluster record: ktok[16] kcell[16] kpcell[16] hdr{klen, rb, re, first pair (global), img_tok}
struct KRec {
    static constexpr int KTOK = 0, KCELL = 16, KPCELL = 32, HDR = 48, WORDS = 56;
};
// Reverse pair record (CSR order of rev_cl):
//   qtok[16] qcell[16] hdr{qlen, class, first, last, key item, global pair index, query item, image * N}
// Record classes (hdr kHFast / kPFast): 1 lattice-fast (window cells iy*kWs+ix),
// 2 medium (one phase, offsets within the global table: packed cells
// (iy+2048)<<16 | (ix+2048)), 0 general (coordinates).
struct PRec {
    static constexpr int QTOK = 0, QCELL = 16, HDR = 32, WORDS = 40;
};
enum { kPQlen = 0, kPFast = 1, kPFirst = 2, kPLast = 3, kPItem = 4, kPIdx = 5, kPQItem = 6, kPImgTok = 7 };
constexpr int kWinC = kRs * kWs + kRs;  // window index of offset (0, 0)
constexpr int kMG = 4 * kMaxHidden + 1;  // tier-3 MLP grad accumulator per head
constexpr int kTabReplicas = 4;          // global tier-2 gradient table copies (spread atomics)

struct AttnParams {
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    const __nv_bfloat16* bk;
    const __nv_bfloat16* bv;
    const float* coords;
    const int32_t* qrec;  // [B*C][QRec::WORDS]
    const int32_t* krec;  // [B*C][KRec::WORDS]
    const int32_t* prec;  // [B*C*G][PRec::WORDS]
    const int32_t* items;       // [2][B*C]: lattice-fast query clusters, then general ones (ascending)
    const int32_t* item_count;  // [2]: fast, general
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
    float2* lsd;    // [B*C, heads, 16] per query-cluster row: {LSE*log2(e), D = rowsum(P o dP)}
                    // (written by the query side, read contiguously by the key side)
    float* dtab_g;  // [kTabReplicas][heads][kWg2] tier-2 gradient (atomics)
    float* part;    // [heads][CTAs][part_width] per-warp gradient partials (of this launch)
    ClusterShape cs;
    int batch;
    int heads;
    int hidden;
    float inv_patch;
    float scale;      // 1/sqrt(d)
    int64_t ldq;      // elements between token rows of q, k, v, dq, dk, dv (heads*d, or 3*heads*d
                      // when the three live interleaved in one [N, 3D] QKV buffer)
    int64_t ldo;      // elements between token rows of out / dout (heads*d)
};
// per-warp partial: window dT [kWs2] | MLP grads [kMG] | blank {dbk[d], dbv[d], dblank}
__host__ __device__ constexpr int part_width(int hd) { return kWs2 + kMG + 2 * hd + 1; }

// ---------------------------------------------------------------- helpers
// Token offset (image * N) of a reverse-pair round.
__device__ __forceinline__ int item_tok(const int32_t* round_rec, const AttnParams&) {
    return round_rec[PRec::HDR + kPImgTok];
}
// Zero a shared-memory range (16-byte granules) with the warp.
__device__ __forceinline__ void zero_shared(void* base, size_t bytes) {
    uint4* p = reinterpret_cast<uint4*>(base);
    for (size_t i = threadIdx.x; i < bytes / 16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
}
// Record words -> shared (16-byte cp.async chunks).
template <int WORDS>
__device__ __forceinline__ void copy_rec(int32_t* dst, const int32_t* src, int lane) {
    static_assert(WORDS % 4 == 0, "record rows are 16-byte multiples");
#pragma unroll
    for (int c = lane; c < WORDS / 4; c += 32) cp_async16(dst + 4 * c, src + 4 * c);
}
// Bias-table window of head h into shared memory, pre-scaled by log2(e), and
// the head's BiasNet MLP parameters (tier 3).
__device__ __forceinline__ void load_head_bias(float* tab, float4* units, const AttnParams& p, int h) {
    for (int e = threadIdx.x; e < kWs2; e += 32) {
        const int oy = e / kWs - kRs, ox = e % kWs - kRs;
        tab[e] = p.tab_g[size_t(h) * kWg2 + (oy + kRg) * kWg + (ox + kRg)] * kLog2e;
    }
    for (int u = threadIdx.x; u < p.hidden; u += 32)
        units[u] = make_float4(p.w1[h * 2 * p.hidden + u], p.w1[h * 2 * p.hidden + p.hidden + u],
                               p.b1[h * p.hidden + u], p.w2[h * p.hidden + u]);
}

// Exact bias (times log2 e) of one pair on a non-fast item: window, global
// table or the BiasNet MLP itself (tiers of attn_common.cuh).
static __device__ __noinline__ float slow_bias2(const AttnParams& p, const float* tab_s,
                                                const float4* units, int h, int64_t img_tok, int qt,
                                                int kt) {
    const float2 qxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + qt);
    const float2 kxy = __ldg(reinterpret_cast<const float2*>(p.coords) + img_tok + kt);
    const TokInfo qi = make_tokinfo(qxy, p.inv_patch), ki = make_tokinfo(kxy, p.inv_patch);
    int gi;
    const int li = lut_index(qi, ki, gi);
    if (li >= 0) return tab_s[li];
    if (gi >= 0) return __ldg(p.tab_g + size_t(h) * kWg2 + gi) * kLog2e;
    return bias_mlp(units, p.hidden, p.b2[h], (kxy.x - qxy.x) * p.inv_patch,
                    (kxy.y - qxy.y) * p.inv_patch) * kLog2e;
}
// ======================================================= swizzled row tiles
// Dense rows of HD bf16 (HD*2 bytes = CPR 16-byte chunks), chunk c of row r
// stored at chunk c ^ sw(r): 8 consecutive rows read at one logical chunk hit
// 8 distinct 16-byte bank groups (ldmatrix / ldmatrix.trans conflict-free
// without padding).  For 8-row-aligned tiles sw(r) depends on r & 7 only, so
// every lane's swizzle term is a per-lane constant.
template <int HD>
struct Swz {
    static constexpr int CPR = HD / 8;                       // chunks per row
    static constexpr int SH = CPR == 8 ? 0 : CPR == 4 ? 1 : 2;  // log2(8 / CPR)
    __device__ static __forceinline__ int sw(int r) { return (r >> SH) & (CPR - 1); }
    // element offset of (row r, logical chunk c)
    __device__ static __forceinline__ int at(int r, int c) { return r * HD + ((c ^ sw(r)) << 3); }
};

template <int HD>
__device__ __forceinline__ void sw_load_a16(uint32_t (&a)[HD / 16][4], const __nv_bfloat16* base, int lane) {
    using S = Swz<HD>;
    const int r = lane & 15;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk)
        ldmatrix_x4(a[kk][0], a[kk][1], a[kk][2], a[kk][3], base + S::at(r, 2 * kk + (lane >> 4)));
}
// s[nt] = A(16 x HD) . B_nt^T; B_nt = rows nt*8.. of `b` (nt < NT-1), or the tile `blast`.
template <int HD, int NT>
__device__ __forceinline__ void sw_mma_abt(float (&s)[NT][4], const uint32_t (&a)[HD / 16][4],
                                           const __nv_bfloat16* b, const __nv_bfloat16* blast, int lane) {
    using S = Swz<HD>;
    const int r = lane & 7;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
        const __nv_bfloat16* kb = nt == NT - 1 ? blast : b + nt * 8 * HD;
        if constexpr (HD >= 32) {
#pragma unroll
            for (int k2 = 0; k2 < HD / 32; ++k2) {
                uint32_t bb[4];
                ldmatrix_x4(bb[0], bb[1], bb[2], bb[3], kb + S::at(r, 4 * k2 + (lane >> 3)));
                mma_bf16_16816(s[nt], a[2 * k2], bb);
                mma_bf16_16816(s[nt], a[2 * k2 + 1], bb + 2);
            }
        } else {
            uint32_t bb[2];
            ldmatrix_x2(bb[0], bb[1], kb + S::at(r, (lane >> 3) & 1));
            mma_bf16_16816(s[nt], a[0], bb);
        }
    }
}
// o += P(16 x 16*KS) . V(rows 0 .. 16*KS-1); P in accumulator layout.
template <int HD, int KS, int NT>
__device__ __forceinline__ void sw_mma_pv(float (&o)[HD / 8][4], const float (&pm)[NT][4],
                                          const __nv_bfloat16* v, int lane) {
    using S = Swz<HD>;
    const int r = lane & 15;
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
            ldmatrix_x4_trans(b[0], b[1], b[2], b[3], v + ks * 16 * HD + S::at(r, nd + (lane >> 4)));
            mma_bf16_16816(o[nd], pa, b);
            mma_bf16_16816(o[nd + 1], pa, b + 2);
        }
    }
}
// Fragments (rows r0 / r0+8) -> swizzled bf16 rows, scaled per row.
template <int HD>
__device__ __forceinline__ void sw_frags_to_rows(__nv_bfloat16* sm, const float (&o)[HD / 8][4], float m0,
                                                 float m1, int lane) {
    using S = Swz<HD>;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        *reinterpret_cast<uint32_t*>(sm + S::at(r0, nd) + c0) = pack_bf16(o[nd][0] * m0, o[nd][1] * m0);
        *reinterpret_cast<uint32_t*>(sm + S::at(r0 + 8, nd) + c0) = pack_bf16(o[nd][2] * m1, o[nd][3] * m1);
    }
}
// Swizzled rows -> global token rows (`g` = row 0 of the image slice, rowbytes
// per token row), 16-byte stores.
template <int HD>
__device__ __forceinline__ void sw_rows_to_global(__nv_bfloat16* g, uint32_t rowbytes, const __nv_bfloat16* sm,
                                                  const int32_t* tok, int nrows, int lane) {
    using S = Swz<HD>;
    constexpr int CPR = S::CPR, RPI = 32 / CPR;
    const int sub = lane / CPR, ch = lane - sub * CPR;
    char* base = reinterpret_cast<char*>(g) + ch * 16;
#pragma unroll
    for (int j = 0; j < 16 / RPI; ++j) {
        const int r = sub + j * RPI;
        if (r < nrows)
            *reinterpret_cast<uint4*>(base + uint32_t(tok[r]) * rowbytes) =
                *reinterpret_cast<const uint4*>(sm + S::at(r, ch));
    }
}
// The same with the lane's row tokens already in registers (tk[j] = token of
// row lane / CPR + j * RPI).
template <int HD>
__device__ __forceinline__ void sw_rows_to_global_t(__nv_bfloat16* g, uint32_t rowbytes, const __nv_bfloat16* sm,
                                                    const int (&tk)[16 / (32 / Swz<HD>::CPR)], int nrows,
                                                    int lane) {
    using S = Swz<HD>;
    constexpr int CPR = S::CPR, RPI = 32 / CPR;
    const int sub = lane / CPR, ch = lane - sub * CPR;
    char* base = reinterpret_cast<char*>(g) + ch * 16;
#pragma unroll
    for (int j = 0; j < 16 / RPI; ++j) {
        const int r = sub + j * RPI;
        if (r < nrows)
            *reinterpret_cast<uint4*>(base + uint32_t(tk[j]) * rowbytes) =
                *reinterpret_cast<const uint4*>(sm + S::at(r, ch));
    }
}
// Gather token rows into a swizzled tile: tile row r <- token tok[r] of the
// image slice at `src` (rowbytes per token row), tok < 0 skipped.  One 32-bit
// multiply-add per row (image slices are < 4 GB).
template <int HD, int NROWS>
__device__ __forceinline__ void sw_gather(__nv_bfloat16* dst, const __nv_bfloat16* src, uint32_t rowbytes,
                                          const int32_t* tok, int lane) {
    using S = Swz<HD>;
    constexpr int CPR = S::CPR, RPI = 32 / CPR, NJ = (NROWS + RPI - 1) / RPI;
    const int sub = lane / CPR, ch = lane - sub * CPR;
    const char* base = reinterpret_cast<const char*>(src) + ch * 16;
    const uint32_t sdst = smem_u32(dst);
    // all token ids first: the cp.async statements are compiler memory barriers, so a token
    // load between two of them would wait out its full shared-memory latency every row
    int t[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int r = sub + j * RPI;
        t[j] = (NROWS % RPI == 0 || r < NROWS) ? tok[r] : -1;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int r = sub + j * RPI;
        if (t[j] >= 0)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst + 2 * S::at(r, ch)),
                         "l"(base + uint32_t(t[j]) * rowbytes)
                         : "memory");
    }
}
// Two tiles gathered by the same token list (Q and dO, or K and V): the ids are loaded once.
template <int HD, int NROWS>
__device__ __forceinline__ void sw_gather2(__nv_bfloat16* dst0, const __nv_bfloat16* src0, uint32_t rowbytes0,
                                           __nv_bfloat16* dst1, const __nv_bfloat16* src1, uint32_t rowbytes1,
                                           const int32_t* tok, int lane) {
    using S = Swz<HD>;
    constexpr int CPR = S::CPR, RPI = 32 / CPR, NJ = (NROWS + RPI - 1) / RPI;
    const int sub = lane / CPR, ch = lane - sub * CPR;
    const char* base0 = reinterpret_cast<const char*>(src0) + ch * 16;
    const char* base1 = reinterpret_cast<const char*>(src1) + ch * 16;
    const uint32_t d0 = smem_u32(dst0), d1 = smem_u32(dst1);
    int t[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int r = sub + j * RPI;
        t[j] = (NROWS % RPI == 0 || r < NROWS) ? tok[r] : -1;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int r = sub + j * RPI;
        if (t[j] >= 0) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d0 + 2 * S::at(r, ch)),
                         "l"(base0 + uint32_t(t[j]) * rowbytes0)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d1 + 2 * S::at(r, ch)),
                         "l"(base1 + uint32_t(t[j]) * rowbytes1)
                         : "memory");
        }
    }
}
// Static blank tile (swizzled): row 0 = blank vector of head h, rows 1..7 zero.
template <int HD>
__device__ __forceinline__ void sw_init_blank_tile(__nv_bfloat16* t, const __nv_bfloat16* blank, int h) {
    for (int i = threadIdx.x; i < 8 * HD; i += 32) t[i] = __float2bfloat16(0.f);
    __syncwarp();
    for (int c = threadIdx.x; c < HD; c += 32) t[Swz<HD>::at(0, c >> 3) + (c & 7)] = blank[h * HD + c];
}

static __device__ __noinline__ float bias_mlp_ool(const float4* units, int hidden, float b2, float ox, float oy) {
    return bias_mlp(units, hidden, b2, ox, oy) * kLog2e;
}
// Bias of the lane's score fragment on a non-fast item (log2 domain): the
// coordinates of the lane's 2 query rows and 2*(NT-1) key slots are loaded
// at once, then each pair takes tier 1 (window) / 2 (global table) / 3 (MLP).
template <int KP, int NT>
__device__ __forceinline__ void slow_bias_frag(float (&s)[NT][4], const int32_t* qtok, const int32_t* ktok,
                                               int nk, const float* tab, const float4* units,
                                               const AttnParams& p, int h, int64_t img_tok, float scale2,
                                               int lane) {
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const float2* xy = reinterpret_cast<const float2*>(p.coords) + img_tok;
    const int qa = qtok[r0] >= 0 ? qtok[r0] : qtok[0], qb = qtok[r0 + 8] >= 0 ? qtok[r0 + 8] : qtok[0];
    const float2 q0 = __ldg(xy + qa), q1 = __ldg(xy + qb);
    float2 kx[KP / 8][2];
#pragma unroll
    for (int nt = 0; nt < KP / 8; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int sl = nt * 8 + c0 + j;
            kx[nt][j] = __ldg(xy + (sl < nk ? ktok[sl] : ktok[0]));
        }
    const TokInfo ti0 = make_tokinfo(q0, p.inv_patch), ti1 = make_tokinfo(q1, p.inv_patch);
    const float* tg = p.tab_g + size_t(h) * kWg2;
#pragma unroll
    for (int nt = 0; nt < KP / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 q = e >= 2 ? q1 : q0, k = kx[nt][e & 1];
            const TokInfo ki = make_tokinfo(k, p.inv_patch);
            int gi;
            const int li = lut_index(e >= 2 ? ti1 : ti0, ki, gi);
            float b;
            if (li >= 0) b = tab[li];
            else if (gi >= 0) b = __ldg(tg + gi) * kLog2e;
            else b = bias_mlp_ool(units, p.hidden, p.b2[h], (k.x - q.x) * p.inv_patch, (k.y - q.y) * p.inv_patch);
            s[nt][e] = fmaf(s[nt][e], scale2, b);
        }
}

// Row stride (floats) of the dS scratch tile: KP + 8 puts the four rows of a
// float2 fragment-store phase in disjoint 8-bank groups (conflict-free).
template <int KP>
constexpr int scr_stride() { return KP + 8; }

// Bias-table gradient of a general (non-fast) item from the row-major dS tile
// `scr` [16][KP]: per query row, lanes walk the key slots (slot lane, lane+32),
// so same-phase keys of one row hit distinct window cells (plain RMW unless
// the record flags duplicate cells); far same-phase pairs go to a global table
// replica (REDG), off-lattice pairs to the MLP partials.
template <int KP>
__device__ __forceinline__ void general_grad_rowpass(const float* scr, const int32_t* qtok, const int32_t* ktok,
                                                     int nk, int qlen, bool dup, float* dtab, float* dtab_rep,
                                                     const float4* units, float* mlpg, const AttnParams& p,
                                                     int64_t img_tok, int lane) {
    const float2* xy = reinterpret_cast<const float2*>(p.coords) + img_tok;
    const bool va = lane < nk, vb = KP > 32 && lane + 32 < nk;
    const float2 ka = __ldg(xy + (va ? ktok[lane] : ktok[0]));
    const float2 kb = __ldg(xy + (vb ? ktok[lane + 32] : ktok[0]));
    const float2 qx = __ldg(xy + (lane < qlen ? qtok[lane] : qtok[0]));
    const TokInfo kia = make_tokinfo(ka, p.inv_patch), kib = make_tokinfo(kb, p.inv_patch);
    for (int r = 0; r < qlen; ++r) {
        const float2 q = make_float2(__shfl_sync(0xffffffffu, qx.x, r), __shfl_sync(0xffffffffu, qx.y, r));
        const TokInfo qi = make_tokinfo(q, p.inv_patch);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const bool v = half ? vb : va;
            const float ds = v ? scr[r * scr_stride<KP>() + lane + 32 * half] : 0.f;
            const TokInfo& ki = half ? kib : kia;
            const float2 k = half ? kb : ka;
            int gi = -1, li = -1;
            if (v) li = lut_index(qi, ki, gi);
            if (v && li >= 0) {
                if (dup) atomicAdd(dtab + li, ds);
                else dtab[li] += ds;
            } else if (v && gi >= 0) {
                atomicAdd(dtab_rep + gi, ds);
            }
            // tier 3 (off-lattice / beyond the table): warp-aggregated MLP gradient
            const bool t3 = v && li < 0 && gi < 0;
            if (__any_sync(0xffffffffu, t3)) {
                const float ox = (k.x - q.x) * p.inv_patch, oy = (k.y - q.y) * p.inv_patch;
                const float d3 = t3 ? ds : 0.f;
                for (int u = 0; u < p.hidden; ++u) {
                    const float4 w = units[u];
                    const float t = tanh_fast(fmaf(w.x, ox, fmaf(w.y, oy, w.z)));
                    const float dpre = d3 * w.w * (1.f - t * t);
                    const float a0 = warp_sum(dpre * ox), a1 = warp_sum(dpre * oy);
                    const float a2 = warp_sum(dpre), a3 = warp_sum(d3 * t);
                    if (lane == 0) {
                        mlpg[u] += a0;
                        mlpg[p.hidden + u] += a1;
                        mlpg[2 * p.hidden + u] += a2;
                        mlpg[3 * p.hidden + u] += a3;
                    }
                }
                const float a4 = warp_sum(d3);
                if (lane == 0) mlpg[4 * p.hidden] += a4;
            }
            __syncwarp();
        }
    }
}

// Bias (log2 domain) of a same-phase pair from packed cells: shared window
// when the offset is inside it, else the global table (L2).
constexpr int kPackC = (kRs << 16) | kRs;
__device__ __forceinline__ int packed_window(int kp, int qp) {
    const int d = kp - qp + kPackC;
    const int lo = d & 0xffff, hi = d >> 16;
    return (unsigned(lo) <= 2u * kRs && unsigned(hi) <= 2u * kRs) ? hi * kWs + lo : -1;
}
__device__ __forceinline__ int packed_global(int kp, int qp) {
    const int dx = (kp & 0xffff) - (qp & 0xffff), dy = (kp >> 16) - (qp >> 16);
    return (dy + kRg) * kWg + dx + kRg;
}
__device__ __forceinline__ float medium_bias2(int kp, int qp, const float* tab, const float* tabg_h) {
    const int li = packed_window(kp, qp);
    return li >= 0 ? tab[li] : __ldg(tabg_h + packed_global(kp, qp)) * kLog2e;
}
template <int KP, int NT>
__device__ __forceinline__ void medium_bias_frag(float (&s)[NT][4], const int32_t* qcell, const int32_t* kcell,
                                                 const float* tab, const float* tabg_h, float scale2, int lane) {
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const int q0 = qcell[r0], q1 = qcell[r0 + 8];
#pragma unroll
    for (int nt = 0; nt < KP / 8; ++nt) {
        const int2 kc = *reinterpret_cast<const int2*>(kcell + nt * 8 + c0);
        s[nt][0] = fmaf(s[nt][0], scale2, medium_bias2(kc.x, q0, tab, tabg_h));
        s[nt][1] = fmaf(s[nt][1], scale2, medium_bias2(kc.y, q0, tab, tabg_h));
        s[nt][2] = fmaf(s[nt][2], scale2, medium_bias2(kc.x, q1, tab, tabg_h));
        s[nt][3] = fmaf(s[nt][3], scale2, medium_bias2(kc.y, q1, tab, tabg_h));
    }
}
// Bias-table gradient of a medium item from the row-major dS tile.
template <int KP>
__device__ __forceinline__ void medium_grad_rowpass(const float* scr, const int32_t* qcell, const int32_t* kcell,
                                                    int nk, int qlen, bool dup, float* dtab, float* rep, int lane) {
    const bool va = lane < nk, vb = KP > 32 && lane + 32 < nk;
    const int ka = va ? kcell[lane] : 0, kb = vb ? kcell[lane + 32] : 0;
    const int qcl = lane < 16 ? qcell[lane] : 0;
    for (int r = 0; r < qlen; ++r) {
        const int qp = __shfl_sync(0xffffffffu, qcl, r);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            if (half ? vb : va) {
                const int kp = half ? kb : ka;
                const float ds = scr[r * scr_stride<KP>() + lane + 32 * half];
                const int li = packed_window(kp, qp);
                if (li >= 0) {
                    if (dup) atomicAdd(dtab + li, ds);
                    else dtab[li] += ds;
                } else {
                    atomicAdd(rep + packed_global(kp, qp), ds);
                }
            }
            __syncwarp();
        }
    }
}

// Masks of the score fragment: padding slots [nk, KP), blank tile (slot KP only).
template <int KP, int NT>
__device__ __forceinline__ void mask_slots(float (&s)[NT][4], int nk, float scale2, float blank2, int lane) {
    const int c0 = 2 * (lane & 3);
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
// Fast-item bias: window lookups by lattice cell difference.
template <int KP, int NT>
__device__ __forceinline__ void fast_bias_frag(float (&s)[NT][4], const int32_t* qcell, const int32_t* kcell,
                                               const float* tab, float scale2, int lane) {
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const int q0 = kWinC - qcell[r0], q1 = kWinC - qcell[r0 + 8];
#pragma unroll
    for (int nt = 0; nt < KP / 8; ++nt) {
        const int2 kc = *reinterpret_cast<const int2*>(kcell + nt * 8 + c0);
        s[nt][0] = fmaf(s[nt][0], scale2, tab[kc.x + q0]);
        s[nt][1] = fmaf(s[nt][1], scale2, tab[kc.y + q0]);
        s[nt][2] = fmaf(s[nt][2], scale2, tab[kc.x + q1]);
        s[nt][3] = fmaf(s[nt][3], scale2, tab[kc.y + q1]);
    }
}

// ======================================================= forward
template <int HD, int KP>
struct FwdCfg {
    static constexpr int NT = KP / 8 + 1;
    static constexpr int QW = QRec<KP>::WORDS;
    struct alignas(16) Smem {
        __nv_bfloat16 Q[16 * HD];
        __nv_bfloat16 K[KP * HD];
        __nv_bfloat16 V[KP * HD];
        __nv_bfloat16 Kb[8 * HD];   // blank key tile
        __nv_bfloat16 O[16 * HD];   // output staging
        int32_t rec[3][QW];
        float tab[kWs2];
        float4 units[kMaxHidden];
    };
};

// Per warp, item i: [Q,K(i) landed] S = QK^T -> issue Q,K(i+1) -> softmax ->
// [V(i) landed] O = PV -> issue V(i+1) -> store O; records two items ahead.
template <int HD, int KP, bool FAST>
__global__ void __launch_bounds__(32, HD >= 64 ? 9 : 14) attn_fwd_kernel(AttnParams p) {
    using C = FwdCfg<HD, KP>;
    using R = QRec<KP>;
    constexpr int NT = C::NT;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
    const int lane = threadIdx.x, h = blockIdx.y;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const int32_t* list = p.items + (FAST ? 0 : p.batch * p.cs.c);
    const int n_items = __ldg(p.item_count + (FAST ? 0 : 1)), stride = gridDim.x;
    const int64_t ld = p.ldq, ldo = p.ldo;
    const uint32_t rowb = uint32_t(ld * 2), rowbo = uint32_t(ldo * 2);
    const __nv_bfloat16* qg = p.q + h * HD;
    const __nv_bfloat16* kg = p.k + h * HD;
    const __nv_bfloat16* vg = p.v + h * HD;

    zero_shared(&sm, sizeof(sm));
    __syncwarp();
    sw_init_blank_tile<HD>(sm.Kb, p.bk, h);
    load_head_bias(sm.tab, sm.units, p, h);
    const float scale2 = p.scale * kLog2e, blank2 = p.blank[h] * kLog2e;
    float bvr[HD / 8][2];
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        bvr[nd][0] = __bfloat162float(p.bv[h * HD + nd * 8 + c0]);
        bvr[nd][1] = __bfloat162float(p.bv[h * HD + nd * 8 + c0 + 1]);
    }
    auto rec_of = [&](int it) -> int32_t* { return sm.rec[it % 3]; };
    // list entries are read one iteration before their record is copied (a dependent global
    // load off the critical path)
    auto list_at = [&](int item) -> int { return item < n_items ? __ldg(list + item) : 0; };
    auto copy_item_rec = [&](int item, int entry, int it) {
        if (item < n_items) copy_rec<C::QW>(rec_of(it), p.qrec + size_t(entry) * C::QW, lane);
    };

    const int i0 = blockIdx.x;
    copy_item_rec(i0, list_at(i0), 0);
    copy_item_rec(i0 + stride, list_at(i0 + stride), 1);
    int next_entry = list_at(i0 + 2 * stride);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    if (i0 < n_items) {
        const int64_t io = int64_t(rec_of(0)[R::HDR + kHImgTok]) * ld;
        sw_gather<HD, 16>(sm.Q, qg + io, rowb, rec_of(0) + R::QTOK, lane);
        sw_gather<HD, KP>(sm.K, kg + io, rowb, rec_of(0) + R::KTOK, lane);
        cp_async_commit();
        sw_gather<HD, KP>(sm.V, vg + io, rowb, rec_of(0) + R::KTOK, lane);
    } else {
        cp_async_commit();
    }
    cp_async_commit();

    int it = 0;
    for (int item = i0; item < n_items; item += stride, ++it) {
        const int i1 = item + stride;
        cp_async_wait<1>();  // Q, K (and record i+1) landed; V may be in flight
        __syncwarp();
        // record fields and the Q fragments before the next record's copy (cp.async is a
        // compiler memory barrier: loads after it would wait out their latency behind it)
        const int32_t* rec = rec_of(it);
        const int32_t* rec1 = rec_of(it + 1);
        const int nk = rec[R::HDR + kHNk], qlen = rec[R::HDR + kHQlen];
        const int64_t img_tok = rec[R::HDR + kHImgTok], io_cur = img_tok * ld;
        const int64_t io_nxt = int64_t(rec1[R::HDR + kHImgTok]) * ld;
        uint32_t qa[HD / 16][4];
        sw_load_a16<HD>(qa, sm.Q, lane);
        copy_item_rec(item + 2 * stride, next_entry, it + 2);
        next_entry = list_at(item + 3 * stride);
        cp_async_commit();
        float s[NT][4];
        sw_mma_abt<HD, NT>(s, qa, sm.K, sm.Kb, lane);
        // the bias lookups (cell ids, table) before the next item's copies: each cp.async is a
        // compiler memory barrier, shared loads behind it would wait on their full latency
        if constexpr (FAST) {
            fast_bias_frag<KP, NT>(s, rec + R::QCELL, rec + R::KCELL, sm.tab, scale2, lane);
        } else {
            if (rec[R::HDR + kHFast] == 2)
                medium_bias_frag<KP, NT>(s, rec + R::QCELL, rec + R::KCELL, sm.tab, p.tab_g + size_t(h) * kWg2,
                                         scale2, lane);
            else
                slow_bias_frag<KP, NT>(s, rec + R::QTOK, rec + R::KTOK, nk, sm.tab, sm.units, p, h, img_tok,
                                       scale2, lane);
        }
        mask_slots<KP, NT>(s, nk, scale2, blank2, lane);
        __syncwarp();  // Q, K consumed: reload them for item i+1
        if (i1 < n_items) {
            sw_gather<HD, 16>(sm.Q, qg + io_nxt, rowb, rec1 + R::QTOK, lane);
            sw_gather<HD, KP>(sm.K, kg + io_nxt, rowb, rec1 + R::KTOK, lane);
        }
        cp_async_commit();

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
        cp_async_wait<2>();  // V(i) landed
        __syncwarp();
        float o[HD / 8][4];
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
        sw_mma_pv<HD, KP / 16, NT>(o, s, sm.V, lane);
        __syncwarp();  // V consumed: reload it for item i+1
        if (i1 < n_items) sw_gather<HD, KP>(sm.V, vg + io_nxt, rowb, rec1 + R::KTOK, lane);
        cp_async_commit();
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
        sw_frags_to_rows<HD>(sm.O, o, 1.f / l0, 1.f / l1, lane);
        if ((lane & 3) == 0) {
            float* lse_img = p.lse + img_tok * p.heads + h;
            if (r0 < qlen) lse_img[uint32_t(rec[R::QTOK + r0]) * uint32_t(p.heads)] = (m0 + __log2f(l0)) * kLn2;
            if (r0 + 8 < qlen) lse_img[uint32_t(rec[R::QTOK + r0 + 8]) * uint32_t(p.heads)] = (m1 + __log2f(l1)) * kLn2;
        }
        __syncwarp();
        sw_rows_to_global<HD>(p.out + img_tok * ldo + h * HD, rowbo, sm.O, rec + R::QTOK, qlen, lane);
    }
    cp_async_wait<0>();
}

// ======================================================= backward, query side
template <int HD, int KP>
struct BwdQCfg {
    static constexpr int NT = KP / 8 + 1;
    static constexpr int kScrFloats = (16 * (KP + 8) > 8 * HD ? 16 * (KP + 8) : 8 * HD);
    static constexpr int QW = QRec<KP>::WORDS;
    struct alignas(16) Smem {
        __nv_bfloat16 Q[16 * HD];
        __nv_bfloat16 dO[16 * HD];
        __nv_bfloat16 K[KP * HD];
        __nv_bfloat16 V[KP * HD];
        __nv_bfloat16 Kb[8 * HD];  // blank key / value tiles
        __nv_bfloat16 Vb[8 * HD];
        float scr[kScrFloats];     // dS tile (bias-table gradient pass) / dQ staging
        float lse[16];
        int32_t rec[3][QW];
        float tab[kWs2];
        float dtab[kWs2];
        float4 units[kMaxHidden];
        float mlpg[kMG];
    };
};

// Per warp, item i (everything of i landed):  S = QK^T, dP = dO.V^T ->
// issue V(i+1) -> P, D, dS -> dQ = dS.K -> issue K(i+1) -> blank grads (Q, dO)
// -> issue Q, dO, LSE(i+1) -> bias-table gradient -> store dQ.
template <int HD, int KP, bool FAST>
__global__ void __launch_bounds__(32, HD >= 64 ? 7 : 11) attn_bwd_q_kernel(AttnParams p) {
    using C = BwdQCfg<HD, KP>;
    using R = QRec<KP>;
    constexpr int NT = C::NT;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
    const int lane = threadIdx.x, h = blockIdx.y;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const int32_t* list = p.items + (FAST ? 0 : p.batch * p.cs.c);
    const int n_items = __ldg(p.item_count + (FAST ? 0 : 1)), stride = gridDim.x;
    const int64_t ld = p.ldq, ldo = p.ldo;
    const uint32_t rowb = uint32_t(ld * 2), rowbo = uint32_t(ldo * 2);
    const __nv_bfloat16* qg = p.q + h * HD;
    const __nv_bfloat16* og = p.dout + h * HD;
    const __nv_bfloat16* kg = p.k + h * HD;
    const __nv_bfloat16* vg = p.v + h * HD;

    zero_shared(&sm, sizeof(sm));
    __syncwarp();
    sw_init_blank_tile<HD>(sm.Kb, p.bk, h);
    sw_init_blank_tile<HD>(sm.Vb, p.bv, h);
    load_head_bias(sm.tab, sm.units, p, h);
    const float scale2 = p.scale * kLog2e, blank2 = p.blank[h] * kLog2e;
    float bkr[HD / 8][2];
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        bkr[nd][0] = __bfloat162float(p.bk[h * HD + nd * 8 + c0]);
        bkr[nd][1] = __bfloat162float(p.bk[h * HD + nd * 8 + c0 + 1]);
    }
    float gbk[HD / 8][2], gbv[HD / 8][2];  // blank grads: row 0 of a rank-1 mma (lanes 0..3)
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) gbk[nd][0] = gbk[nd][1] = gbv[nd][0] = gbv[nd][1] = 0.f;
    float gblank = 0.f;

    auto list_at = [&](int item) -> int { return item < n_items ? __ldg(list + item) : 0; };
    auto copy_item_rec = [&](int item, int entry, int32_t* dst) {
        if (item < n_items) copy_rec<C::QW>(dst, p.qrec + size_t(entry) * C::QW, lane);
    };
    auto issue_qo = [&](const int32_t* rec, int64_t img_tok) {
        sw_gather2<HD, 16>(sm.Q, qg + img_tok * ld, rowb, sm.dO, og + img_tok * ldo, rowbo, rec + R::QTOK, lane);
        if (lane < 16) {
            const int qt = rec[R::QTOK + lane];
            if (qt >= 0) cp_async4(sm.lse + lane, p.lse + (img_tok + qt) * p.heads + h);
            else sm.lse[lane] = INFINITY;
        }
    };

    const int i0 = blockIdx.x;
    int rc = 0;  // ring slot of the current item's record
    copy_item_rec(i0, list_at(i0), sm.rec[0]);
    copy_item_rec(i0 + stride, list_at(i0 + stride), sm.rec[1]);
    int next_entry = list_at(i0 + 2 * stride);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    if (i0 < n_items) {
        const int64_t it0 = sm.rec[0][R::HDR + kHImgTok];
        issue_qo(sm.rec[0], it0);
        sw_gather2<HD, KP>(sm.K, kg + it0 * ld, rowb, sm.V, vg + it0 * ld, rowb, sm.rec[0] + R::KTOK, lane);
    }
    cp_async_commit();

    float* dtab = sm.dtab;
    for (int item = i0; item < n_items; item += stride) {
        const int r1 = rc == 2 ? 0 : rc + 1, r2 = r1 == 2 ? 0 : r1 + 1;
        cp_async_wait<0>();  // rows of this item and the record of the next one landed
        __syncwarp();
        // record fields and the Q / dO fragments before the next record's copy (see the forward)
        const int32_t* rec = sm.rec[rc];
        const int32_t* rec1 = sm.rec[r1];
        const bool more = item + stride < n_items;
        const int nk = rec[R::HDR + kHNk], qlen = rec[R::HDR + kHQlen];
        const int64_t img_tok = rec[R::HDR + kHImgTok];
        const int64_t nxt_tok = rec1[R::HDR + kHImgTok];
        uint32_t qa[HD / 16][4], oa[HD / 16][4];
        sw_load_a16<HD>(qa, sm.Q, lane);
        sw_load_a16<HD>(oa, sm.dO, lane);
        copy_item_rec(item + 2 * stride, next_entry, sm.rec[r2]);
        next_entry = list_at(item + 3 * stride);
        cp_async_commit();
        float s[NT][4], dp[NT][4];
        sw_mma_abt<HD, NT>(s, qa, sm.K, sm.Kb, lane);
        sw_mma_abt<HD, NT>(dp, oa, sm.V, sm.Vb, lane);
        // bias lookups and LSE before the next item's V copies (cp.async = compiler memory barrier)
        const int cls = rec[R::HDR + kHFast];
        if constexpr (FAST) {
            fast_bias_frag<KP, NT>(s, rec + R::QCELL, rec + R::KCELL, sm.tab, scale2, lane);
        } else {
            if (cls == 2)
                medium_bias_frag<KP, NT>(s, rec + R::QCELL, rec + R::KCELL, sm.tab, p.tab_g + size_t(h) * kWg2,
                                         scale2, lane);
            else
                slow_bias_frag<KP, NT>(s, rec + R::QTOK, rec + R::KTOK, nk, sm.tab, sm.units, p, h, img_tok,
                                       scale2, lane);
        }
        mask_slots<KP, NT>(s, nk, scale2, blank2, lane);
        const float ls0 = sm.lse[r0] * kLog2e, ls1 = sm.lse[r0 + 8] * kLog2e;
        __syncwarp();  // V consumed
        if (more) sw_gather<HD, KP>(sm.V, vg + nxt_tok * ld, rowb, rec1 + R::KTOK, lane);
        cp_async_commit();

        // P = exp(S - LSE);  D = rowsum(P o dP)
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
        if ((lane & 3) == 0) {  // padding rows get {+inf, 0}: P = 0 on the key side
            float2* l = p.lsd + (size_t(rec[R::HDR + kHItem]) * p.heads + h) * 16;
            l[r0] = r0 < qlen ? make_float2(ls0, D0) : make_float2(INFINITY, 0.f);
            l[r0 + 8] = r0 + 8 < qlen ? make_float2(ls1, D1) : make_float2(INFINITY, 0.f);
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
        // ---- dQ = dS . K / sqrt(d)  (+ blank rank-1 dS_b x blank_k)
        float dqa[HD / 8][4];
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) dqa[nd][0] = dqa[nd][1] = dqa[nd][2] = dqa[nd][3] = 0.f;
        sw_mma_pv<HD, KP / 16, NT>(dqa, s, sm.K, lane);
        __syncwarp();  // K consumed
        if (more) sw_gather<HD, KP>(sm.K, kg + nxt_tok * ld, rowb, rec1 + R::KTOK, lane);
        cp_async_commit();
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
            using S = Swz<HD>;
            const int rr = lane & 15;
#pragma unroll
            for (int nd = 0; nd < HD / 8; nd += 2) {
                uint32_t b[4], bo[4];
                ldmatrix_x4_trans(b[0], b[1], b[2], b[3], sm.Q + S::at(rr, nd + (lane >> 4)));
                ldmatrix_x4_trans(bo[0], bo[1], bo[2], bo[3], sm.dO + S::at(rr, nd + (lane >> 4)));
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
        __syncwarp();  // Q, dO, LSE consumed
        if (more) issue_qo(rec1, nxt_tok);
        cp_async_commit();
        // ---- bias-table gradient (dS tile row-major in scratch, then one pass per query row)
        float* scr = sm.scr;
        constexpr int SS = scr_stride<KP>();
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) {
            *reinterpret_cast<float2*>(scr + r0 * SS + nt * 8 + c0) = make_float2(s[nt][0], s[nt][1]);
            *reinterpret_cast<float2*>(scr + (r0 + 8) * SS + nt * 8 + c0) = make_float2(s[nt][2], s[nt][3]);
        }
        __syncwarp();
        const bool dup = (rec[R::HDR + kHDup0] | rec[R::HDR + kHDup1]) != 0;
        if constexpr (FAST) {
            // Rows of one query hold pairwise-distinct key cells, so lanes over the
            // key slots of one row write distinct window entries: plain RMW
            // (duplicate key coordinates -> the record flags force atomics).
            const bool va = lane < nk, vb = KP > 32 && lane + 32 < nk;
            float* da = dtab + (va ? rec[R::KCELL + lane] + kWinC : 0);
            float* db = dtab + (vb ? rec[R::KCELL + lane + 32] + kWinC : 0);
            const int qcl = lane < 16 ? rec[R::QCELL + lane] : 0;
            if (!dup) {
                for (int r = 0; r < qlen; ++r) {
                    const int qc = __shfl_sync(0xffffffffu, qcl, r);
                    if (va) da[-qc] += scr[r * SS + lane];
                    if (vb) db[-qc] += scr[r * SS + lane + 32];
                    __syncwarp();
                }
            } else {
                for (int r = 0; r < qlen; ++r) {
                    const int qc = __shfl_sync(0xffffffffu, qcl, r);
                    if (va) atomicAdd(da - qc, scr[r * SS + lane]);
                    __syncwarp();
                    if (vb) atomicAdd(db - qc, scr[r * SS + lane + 32]);
                    __syncwarp();
                }
            }
        } else {
            float* rep = p.dtab_g + (size_t(blockIdx.x & (kTabReplicas - 1)) * p.heads + h) * kWg2;
            if (cls == 2)
                medium_grad_rowpass<KP>(scr, rec + R::QCELL, rec + R::KCELL, nk, qlen, dup, dtab, rep, lane);
            else
                general_grad_rowpass<KP>(scr, rec + R::QTOK, rec + R::KTOK, nk, qlen, dup, dtab, rep, sm.units,
                                         sm.mlpg, p, img_tok, lane);
        }
        __syncwarp();
        // ---- store dQ (staged through the scratch)
        __nv_bfloat16* Ost = reinterpret_cast<__nv_bfloat16*>(scr);
        sw_frags_to_rows<HD>(Ost, dqa, p.scale, p.scale, lane);
        __syncwarp();
        sw_rows_to_global<HD>(p.dq + img_tok * ld + h * HD, rowb, Ost, rec + R::QTOK, qlen, lane);
        __syncwarp();
        rc = r1;
    }
    cp_async_wait<0>();

    // ---- per-warp partials (reduced in a fixed order by attn_part_reduce_kernel)
    __syncwarp();
    float* part = p.part + (size_t(h) * gridDim.x + blockIdx.x) * part_width(HD);
    for (int i = lane; i < kWs2; i += 32) part[i] = dtab[i];
    for (int i = lane; i < kMG; i += 32) part[kWs2 + i] = sm.mlpg[i];
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
// One pipeline round = one reverse pair (key cluster c', query cluster c).
template <int HD>
struct BwdKCfg {
    static constexpr int RECW = PRec::WORDS + KRec::WORDS;  // pair record | key record
    struct alignas(16) Smem {
        __nv_bfloat16 Q[2][16 * HD];   // per round (double-buffered)
        __nv_bfloat16 dO[2][16 * HD];
        __nv_bfloat16 K[16 * HD];      // first round of a key cluster
        __nv_bfloat16 V[16 * HD];
        __nv_bfloat16 dK[16 * HD];     // output staging (last round)
        __nv_bfloat16 dV[16 * HD];
        float2 lsd[2][16];             // {LSE*log2(e), D} of the round's query rows
        int32_t rec[3][RECW];
        float tab[kWs2];
        float4 units[kMaxHidden];
    };
};

// Per warp, round r (everything of r landed): [first: K, V -> registers] ->
// issue record r+2 and the rows of round r+1 -> S^T = K Q^T, dP^T = V dO^T ->
// P^T, dS^T -> dV += P^T dO, dK += dS^T Q -> [last: store dK, dV].
template <int HD>
__global__ void __launch_bounds__(32, HD >= 64 ? 9 : 16) attn_bwd_kv_kernel(AttnParams p) {
    using C = BwdKCfg<HD>;
    constexpr int KR = PRec::WORDS;  // key record offset inside a round record
    extern __shared__ __align__(128) uint8_t smem_raw[];
    auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
    const int lane = threadIdx.x, h = blockIdx.y;
    const int r0 = lane >> 2, c0 = 2 * (lane & 3);
    const int n_items = p.batch * p.cs.c, stride = gridDim.x;
    const int64_t ld = p.ldq, ldo = p.ldo;
    const uint32_t rowb = uint32_t(ld * 2), rowbo = uint32_t(ldo * 2);
    using S = Swz<HD>;

    zero_shared(&sm, sizeof(sm));
    __syncwarp();
    load_head_bias(sm.tab, sm.units, p, h);
    const float scale2 = p.scale * kLog2e;

    // Round cursor: global pair index of a round, -1 past the end.
    auto first_pair = [&](int item) -> int {
        return item < n_items ? __ldg(p.krec + size_t(item) * KRec::WORDS + KRec::HDR + 3) : -1;
    };
    // the key record only rides along with the first round of its cluster
    auto copy_round = [&](int pair, int item, bool with_krec, int32_t* dst) {
        if (pair < 0) return;
        copy_rec<PRec::WORDS>(dst, p.prec + size_t(pair) * PRec::WORDS, lane);
        if (with_krec) copy_rec<KRec::WORDS>(dst + KR, p.krec + size_t(item) * KRec::WORDS, lane);
    };
    // Round after the round whose record is `rec` (landed): the next pair of the
    // same key cluster, else the first pair of the cluster `stride` further on
    // (nx_first, prefetched one cluster ahead).
    int nx_first = -1;
    auto advance = [&](const int32_t* rec, int& item, bool& newc) -> int {
        item = rec[PRec::HDR + kPItem];
        newc = rec[PRec::HDR + kPLast] != 0;
        if (!newc) return rec[PRec::HDR + kPIdx] + 1;
        const int r = nx_first;
        item += stride;
        nx_first = first_pair(item + stride);
        return r;
    };
    auto issue_rows = [&](int buf, const int32_t* rec) {
        const int64_t img_tok = int64_t(item_tok(rec, p));
        const int64_t base = img_tok * ld + h * HD;
        // record fields read before the copies (each cp.async is a compiler memory barrier)
        const bool first = rec[PRec::HDR + kPFirst] != 0;
        const float2* lsd_src = p.lsd + (size_t(rec[PRec::HDR + kPQItem]) * p.heads + h) * 16 + 2 * lane;
        if (lane < 8) cp_async16(sm.lsd[buf] + 2 * lane, lsd_src);
        sw_gather2<HD, 16>(sm.Q[buf], p.q + base, rowb, sm.dO[buf], p.dout + img_tok * ldo + h * HD, rowbo,
                           rec + PRec::QTOK, lane);
        if (first)
            sw_gather2<HD, 16>(sm.K, p.k + base, rowb, sm.V, p.v + base, rowb, rec + KR + KRec::KTOK, lane);
    };

    // prologue: records of rounds 0 and 1, rows of round 0
    int pr0 = first_pair(blockIdx.x), it1 = 0;
    nx_first = first_pair(blockIdx.x + stride);
    copy_round(pr0, blockIdx.x, true, sm.rec[0]);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    bool nc1 = false;
    int pr1 = pr0 >= 0 ? advance(sm.rec[0], it1, nc1) : -1;
    copy_round(pr1, it1, nc1, sm.rec[1]);
    if (pr0 >= 0) issue_rows(0, sm.rec[0]);
    cp_async_commit();

    uint32_t ka[HD / 16][4], va[HD / 16][4];
    float dk[HD / 8][4], dv[HD / 8][4];
    int kq0 = 0, kq1 = 0, kt0 = 0, kt1 = 0, kp0 = 0, kp1 = 0, klen = 0;
    constexpr int SRPI = 32 / Swz<HD>::CPR;  // rows per dK/dV store instruction
    int stok[16 / SRPI];                      // key tokens of the lane's store rows
    const float* tabg_h = p.tab_g + size_t(h) * kWg2;
    int rc = 0;
    for (int it = 0; pr0 >= 0; ++it) {
        const int r1 = rc == 2 ? 0 : rc + 1, r2 = r1 == 2 ? 0 : r1 + 1;
        const int buf = it & 1;
        cp_async_wait<0>();  // rows of round it, record of round it+1
        __syncwarp();
        const int32_t* rec = sm.rec[rc];
        const int32_t* krec = rec + KR;
        const bool first = rec[PRec::HDR + kPFirst] != 0, last = rec[PRec::HDR + kPLast] != 0;
        const int64_t img_tok = item_tok(rec, p);
        if (first) {
            sw_load_a16<HD>(ka, sm.K, lane);
            sw_load_a16<HD>(va, sm.V, lane);
#pragma unroll
            for (int nd = 0; nd < HD / 8; ++nd)
#pragma unroll
                for (int e = 0; e < 4; ++e) dk[nd][e] = dv[nd][e] = 0.f;
            klen = krec[KRec::HDR];
#pragma unroll
            for (int j = 0; j < 16 / SRPI; ++j) stok[j] = krec[KRec::KTOK + lane / Swz<HD>::CPR + j * SRPI];
            kq0 = krec[KRec::KCELL + r0] + kWinC;
            kq1 = krec[KRec::KCELL + r0 + 8] + kWinC;
            kt0 = krec[KRec::KTOK + (r0 < klen ? r0 : 0)];
            kt1 = krec[KRec::KTOK + (r0 + 8 < klen ? r0 + 8 : 0)];
            kp0 = krec[KRec::KPCELL + r0];
            kp1 = krec[KRec::KPCELL + r0 + 8];
            __syncwarp();  // K, V consumed
        }
        int it2 = 0;
        bool nc2 = false;
        const int pr2 = pr1 >= 0 ? advance(sm.rec[r1], it2, nc2) : -1;
        copy_round(pr2, it2, nc2, sm.rec[r2]);
        if (pr1 >= 0) issue_rows(buf ^ 1, sm.rec[r1]);
        cp_async_commit();

        const __nv_bfloat16* Qb = sm.Q[buf];
        const __nv_bfloat16* Ob = sm.dO[buf];
        float sT[2][4], dpT[2][4];
        sw_mma_abt<HD, 2>(sT, ka, Qb, Qb + 8 * HD, lane);
        sw_mma_abt<HD, 2>(dpT, va, Ob, Ob + 8 * HD, lane);
        const int pcls = rec[PRec::HDR + kPFast];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int qc = nt * 8 + c0;
            float b[4];
            if (pcls == 2) {
                const int2 qcl = *reinterpret_cast<const int2*>(rec + PRec::QCELL + qc);
                b[0] = medium_bias2(kp0, qcl.x, sm.tab, tabg_h);
                b[1] = medium_bias2(kp0, qcl.y, sm.tab, tabg_h);
                b[2] = medium_bias2(kp1, qcl.x, sm.tab, tabg_h);
                b[3] = medium_bias2(kp1, qcl.y, sm.tab, tabg_h);
            } else if (pcls == 1) {
                const int2 qcl = *reinterpret_cast<const int2*>(rec + PRec::QCELL + qc);
                b[0] = sm.tab[kq0 - qcl.x];
                b[1] = sm.tab[kq0 - qcl.y];
                b[2] = sm.tab[kq1 - qcl.x];
                b[3] = sm.tab[kq1 - qcl.y];
            } else {
                const int qlen = rec[PRec::HDR + kPQlen];
                const int qa = rec[PRec::QTOK + (qc < qlen ? qc : 0)];
                const int qb = rec[PRec::QTOK + (qc + 1 < qlen ? qc + 1 : 0)];
                b[0] = slow_bias2(p, sm.tab, sm.units, h, img_tok, qa, kt0);
                b[1] = slow_bias2(p, sm.tab, sm.units, h, img_tok, qb, kt0);
                b[2] = slow_bias2(p, sm.tab, sm.units, h, img_tok, qa, kt1);
                b[3] = slow_bias2(p, sm.tab, sm.units, h, img_tok, qb, kt1);
            }
            const float4 ld4 = *reinterpret_cast<const float4*>(sm.lsd[buf] + qc);  // rows qc, qc+1
            const float lv[4] = {ld4.x, ld4.z, ld4.x, ld4.z};
            const float dvv[4] = {ld4.y, ld4.w, ld4.y, ld4.w};
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
        const int rr = lane & 15;
#pragma unroll
        for (int nd = 0; nd < HD / 8; nd += 2) {
            uint32_t b[4], bq[4];
            ldmatrix_x4_trans(b[0], b[1], b[2], b[3], Ob + S::at(rr, nd + (lane >> 4)));
            ldmatrix_x4_trans(bq[0], bq[1], bq[2], bq[3], Qb + S::at(rr, nd + (lane >> 4)));
            mma_bf16_16816(dv[nd], pa, b);
            mma_bf16_16816(dv[nd + 1], pa, b + 2);
            mma_bf16_16816(dk[nd], da, bq);
            mma_bf16_16816(dk[nd + 1], da, bq + 2);
        }
        if (last) {
            sw_frags_to_rows<HD>(sm.dK, dk, p.scale, p.scale, lane);
            sw_frags_to_rows<HD>(sm.dV, dv, 1.f, 1.f, lane);
            __syncwarp();
            sw_rows_to_global_t<HD>(p.dk + img_tok * ld + h * HD, rowb, sm.dK, stok, klen, lane);
            sw_rows_to_global_t<HD>(p.dv + img_tok * ld + h * HD, rowb, sm.dV, stok, klen, lane);
            __syncwarp();
        }
        pr0 = pr1;
        pr1 = pr2;
        rc = r1;
    }
    cp_async_wait<0>();
}

// ------------------------------------------------------------ launchers
template <typename K>
inline int persistent_grid(K kern, size_t smem, int items, int heads, dim3& grid) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
    }
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem);
    if (e != cudaSuccess) return cuda_status(e, "occupancy");
    if (occ < 1) return fail(AFFMAE_EUNSUPPORTED, "attention: kernel does not fit on an SM");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = kNumSMs;
    const int per_head = std::max(1, std::min(occ * sms / heads, kMaxCtasPerGroup));
    grid = dim3(unsigned(std::min(items, per_head)), unsigned(heads), 1);
    return AFFMAE_OK;
}

// Two launches per pass: the lattice-fast item list on the caller's stream and,
// concurrently, the general list (7-9 % of the clusters at 256^2 grids, but the
// long items: launched first so they start early; a smaller grid measured slower) on a per-thread side stream forked and joined
// with events -- capture-safe, so both land in the caller's CUDA graph.  Item
// counts live on the device, so the launch shapes are static.
struct ForkStream {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    int init() {
        if (side) return AFFMAE_OK;
        AFFMAE_CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        AFFMAE_CUDA_CHECK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        AFFMAE_CUDA_CHECK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
        return AFFMAE_OK;
    }
};
// one side stream per (host thread, device): streams are bound to the device
// current at creation
inline ForkStream* fork_stream() {
    static thread_local ForkStream f[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    return &f[dev];
}
template <typename LaunchMain, typename LaunchSide>
inline int launch_forked(cudaStream_t st, LaunchSide side_fn, LaunchMain main_fn) {
    ForkStream* fp = fork_stream();
    if (!fp) return fail(AFFMAE_ECUDA, "attention: cudaGetDevice");
    ForkStream& f = *fp;
    int rc = f.init();
    if (rc) return rc;
    AFFMAE_CUDA_CHECK(cudaEventRecord(f.fork, st));
    AFFMAE_CUDA_CHECK(cudaStreamWaitEvent(f.side, f.fork, 0));
    if ((rc = side_fn(f.side))) return rc;
    AFFMAE_CUDA_CHECK(cudaEventRecord(f.join, f.side));
    if ((rc = main_fn(st))) return rc;
    AFFMAE_CUDA_CHECK(cudaStreamWaitEvent(st, f.join, 0));
    return AFFMAE_OK;
}

template <int HD, int KP>
int launch_fwd(const AttnParams& p, cudaStream_t st) {
    auto kf = attn_fwd_kernel<HD, KP, true>;
    auto kg = attn_fwd_kernel<HD, KP, false>;
    const size_t smem = sizeof(typename FwdCfg<HD, KP>::Smem);
    dim3 gf, gg;
    int rc = persistent_grid(kf, smem, p.batch * p.cs.c, p.heads, gf);
    if (rc) return rc;
    if ((rc = persistent_grid(kg, smem, p.batch * p.cs.c, p.heads, gg))) return rc;
    return launch_forked(
        st,
        [&](cudaStream_t s) {
            kg<<<gg, 32, smem, s>>>(p);
            AFFMAE_LAUNCH_CHECK("attn_fwd_kernel<general>");
            return AFFMAE_OK;
        },
        [&](cudaStream_t s) {
            kf<<<gf, 32, smem, s>>>(p);
            AFFMAE_LAUNCH_CHECK("attn_fwd_kernel<fast>");
            return AFFMAE_OK;
        });
}

// Launches the query-side kernels; `grid_x[2]` returns their CTA counts per
// head; their per-warp partials go to part and part + heads*grid_x[0]*part_width.
template <int HD, int KP>
int launch_bwd_q(const AttnParams& p, cudaStream_t st, int* grid_x) {
    auto kf = attn_bwd_q_kernel<HD, KP, true>;
    auto kg = attn_bwd_q_kernel<HD, KP, false>;
    const size_t smem = sizeof(typename BwdQCfg<HD, KP>::Smem);
    dim3 gf, gg;
    int rc = persistent_grid(kf, smem, p.batch * p.cs.c, p.heads, gf);
    if (rc) return rc;
    if ((rc = persistent_grid(kg, smem, p.batch * p.cs.c, p.heads, gg))) return rc;
    grid_x[0] = int(gf.x);
    grid_x[1] = int(gg.x);
    AttnParams q = p;
    q.part = p.part + size_t(p.heads) * grid_x[0] * part_width(HD);
    return launch_forked(
        st,
        [&](cudaStream_t s) {
            kg<<<gg, 32, smem, s>>>(q);
            AFFMAE_LAUNCH_CHECK("attn_bwd_q_kernel<general>");
            return AFFMAE_OK;
        },
        [&](cudaStream_t s) {
            kf<<<gf, 32, smem, s>>>(p);
            AFFMAE_LAUNCH_CHECK("attn_bwd_q_kernel<fast>");
            return AFFMAE_OK;
        });
}

template <int HD>
int launch_bwd_kv(const AttnParams& p, cudaStream_t st) {
    auto kern = attn_bwd_kv_kernel<HD>;
    const size_t smem = sizeof(typename BwdKCfg<HD>::Smem);
    dim3 grid;
    int rc = persistent_grid(kern, smem, p.batch * p.cs.c, p.heads, grid);
    if (rc) return rc;
    kern<<<grid, 32, smem, st>>>(p);
    AFFMAE_LAUNCH_CHECK("attn_bwd_kv_kernel");
    return AFFMAE_OK;
}

#define AFFMAE_INSTANTIATE_ATTN_QK(HD_, KP_)                               \
    template int launch_fwd<HD_, KP_>(const AttnParams&, cudaStream_t); \
    template int launch_bwd_q<HD_, KP_>(const AttnParams&, cudaStream_t, int*);
#define AFFMAE_INSTANTIATE_ATTN_KV(HD_) template int launch_bwd_kv<HD_>(const AttnParams&, cudaStream_t);

}  // namespace affmae_b200
