// Host side of the cluster attention: validation, workspace layout, BiasNet
// table build, the per-call plan records the kernels stream through, kernel
// variant dispatch and the (fixed-order) gradient finalisation.
// Kernels: attn_kernels.cuh (instantiated per head_dim in attn_inst_d*.cu).
#include <climits>
#include <cstdlib>

#include "attn_kernels.cuh"

namespace affmae_b200 {

constexpr int kFinBlocks = 64;  // blocks per head of the BiasNet-gradient finalize pass

// ------------------------------------------------------------ bias table
// T[h][(oy+kRg)*kWg + (ox+kRg)] = b2 + sum_u w2 tanh(w1x ox + w1y oy + b1)
// (BiasNet::eval at integer patch offsets, proj/src/attention.cpp:33-42).
// Only the box |offset| <= R of the table is ever read, R = max(plan radius,
// window radius): the plan records the largest pair offset of its items.
__device__ __forceinline__ int used_radius(const int32_t* rmax) {
    const int r = *rmax;
    return r < kRs ? kRs : (r > kRg ? kRg : r);
}
__global__ void bias_table_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                  const float* __restrict__ w2, const float* __restrict__ b2,
                                  int heads, int hidden, const int32_t* __restrict__ rmax,
                                  float* __restrict__ tab) {
    const int R = used_radius(rmax), side = 2 * R + 1, box = side * side;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < heads * box; i += gridDim.x * blockDim.x) {
        const int h = i / box, e = i - h * box;
        const int oy = e / side - R, ox = e - (e / side) * side - R;
        float acc = b2[h];
        for (int u = 0; u < hidden; ++u) {
            const float pre = w1[h * 2 * hidden + u] * float(ox) + w1[h * 2 * hidden + hidden + u] * float(oy) +
                              b1[h * hidden + u];
            acc += w2[h * hidden + u] * tanhf(pre);
        }
        tab[size_t(h) * kWg2 + (oy + kRg) * kWg + (ox + kRg)] = acc;
    }
}
// zero the used box of every replica of the table gradient
__global__ void dtab_zero_kernel(float* __restrict__ dtab, int heads, const int32_t* __restrict__ rmax) {
    const int R = used_radius(rmax), side = 2 * R + 1, box = side * side;
    const int n = kTabReplicas * heads * box;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int rh = i / box, e = i - rh * box;
        const int oy = e / side - R, ox = e - (e / side) * side - R;
        dtab[size_t(rh) * kWg2 + (oy + kRg) * kWg + (ox + kRg)] = 0.f;
    }
}

// -------------------------------------------------------------- plan records
// Lattice cell of a token (window coordinates): iy * kWs + ix.  Two tokens of
// one phase have window offset kcell - qcell == (dy * kWs + dx).
__device__ __forceinline__ int tok_cell(const TokInfo& t) { return t.iy * kWs + t.ix; }
// Packed lattice cell (iy + 2048) << 16 | (ix + 2048) of a "medium" record (attn_kernels.cuh).
__device__ __forceinline__ int tok_pcell(const TokInfo& t) { return ((t.iy + 2048) << 16) | (t.ix + 2048); }
__device__ __forceinline__ bool pcell_ok(const TokInfo& t) {
    return unsigned(t.ix + 2048) < 4096u && unsigned(t.iy + 2048) < 4096u;
}

struct Bbox {
    int xmin, xmax, ymin, ymax;
};
__device__ __forceinline__ Bbox warp_bbox(bool valid, const TokInfo& t) {
    Bbox b;
    b.xmin = __reduce_min_sync(0xffffffffu, valid ? t.ix : INT_MAX);
    b.xmax = __reduce_max_sync(0xffffffffu, valid ? t.ix : INT_MIN);
    b.ymin = __reduce_min_sync(0xffffffffu, valid ? t.iy : INT_MAX);
    b.ymax = __reduce_max_sync(0xffffffffu, valid ? t.iy : INT_MIN);
    return b;
}
__device__ __forceinline__ bool bbox_fits(const Bbox& q, const Bbox& k) {
    // every key-minus-query offset inside [-kRs, kRs]^2 (64-bit: no overflow on far tokens)
    return int64_t(k.xmax) - q.xmin <= kRs && int64_t(q.xmax) - k.xmin <= kRs &&
           int64_t(k.ymax) - q.ymin <= kRs && int64_t(q.ymax) - k.ymin <= kRs;
}
__device__ __forceinline__ bool bbox_fits_r(const Bbox& q, const Bbox& k, int r) {
    return int64_t(k.xmax) - q.xmin <= r && int64_t(q.xmax) - k.xmin <= r &&
           int64_t(k.ymax) - q.ymin <= r && int64_t(q.ymax) - k.ymin <= r;
}
__device__ __forceinline__ bool warp_one_phase(bool valid, const TokInfo& t) {
    const uint32_t fx0 = __reduce_min_sync(0xffffffffu, valid ? t.fx : 0xffffffffu);
    const uint32_t fx1 = __reduce_max_sync(0xffffffffu, valid ? t.fx : 0u);
    const uint32_t fy0 = __reduce_min_sync(0xffffffffu, valid ? t.fy : 0xffffffffu);
    const uint32_t fy1 = __reduce_max_sync(0xffffffffu, valid ? t.fy : 0u);
    return fx0 == fx1 && fy0 == fy1;
}
// Bounding boxes / phase of up to two warp-chunks of tokens combined.
struct TokAgg {
    int qx0 = INT_MAX, qx1 = INT_MIN, qy0 = INT_MAX, qy1 = INT_MIN;
    int kx0 = INT_MAX, kx1 = INT_MIN, ky0 = INT_MAX, ky1 = INT_MIN;
    uint32_t fx0 = 0xffffffffu, fx1 = 0, fy0 = 0xffffffffu, fy1 = 0;
    __device__ void add(const TokInfo& t, bool is_key) {
        if (is_key) {
            kx0 = min(kx0, t.ix); kx1 = max(kx1, t.ix); ky0 = min(ky0, t.iy); ky1 = max(ky1, t.iy);
        } else {
            qx0 = min(qx0, t.ix); qx1 = max(qx1, t.ix); qy0 = min(qy0, t.iy); qy1 = max(qy1, t.iy);
        }
        fx0 = min(fx0, t.fx); fx1 = max(fx1, t.fx); fy0 = min(fy0, t.fy); fy1 = max(fy1, t.fy);
    }
    bool far = false;  // a token outside the packed-cell range
    // 1: lattice-fast (one phase, offsets inside the shared window); 2: medium
    // (one phase, offsets inside the global table); 0: general.
    __device__ int cls(int* radius) const {
        Bbox q{__reduce_min_sync(0xffffffffu, qx0), __reduce_max_sync(0xffffffffu, qx1),
               __reduce_min_sync(0xffffffffu, qy0), __reduce_max_sync(0xffffffffu, qy1)};
        Bbox k{__reduce_min_sync(0xffffffffu, kx0), __reduce_max_sync(0xffffffffu, kx1),
               __reduce_min_sync(0xffffffffu, ky0), __reduce_max_sync(0xffffffffu, ky1)};
        {   // largest |key - query| offset along either axis
            int64_t rr = int64_t(k.xmax) - q.xmin;
            rr = max(rr, int64_t(q.xmax) - k.xmin);
            rr = max(rr, int64_t(k.ymax) - q.ymin);
            rr = max(rr, int64_t(q.ymax) - k.ymin);
            *radius = int(min(max(rr, int64_t(0)), int64_t(kRg)));
        }
        const bool ph = __reduce_min_sync(0xffffffffu, fx0) == __reduce_max_sync(0xffffffffu, fx1) &&
                        __reduce_min_sync(0xffffffffu, fy0) == __reduce_max_sync(0xffffffffu, fy1);
        const bool anyfar = __any_sync(0xffffffffu, far);
        if (!ph) return 0;
        if (bbox_fits(q, k)) return 1;
        return !anyfar && bbox_fits_r(q, k, kRg) ? 2 : 0;
    }
};

// Query-cluster records (one warp per (image, cluster)): query tokens, the
// key token of every neighbourhood slot in reference order
// (cluster_neighborhood, proj/src/geometry.cpp:173-183; lattice-fast items
// permute it, see below), lattice cells, nk,
// qlen, the lattice-fast flag and duplicate-cell flags of the two key halves.
template <int KP>
__global__ void attn_qrec_kernel(const float* __restrict__ coords, const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ nbr_cl, ClusterShape cs, int64_t items,
                                 float inv_patch, int32_t* __restrict__ qrec, int32_t* __restrict__ rmax) {
    using R = QRec<KP>;
    static_assert(KP <= 64, "two key slots per lane");
    constexpr int E = 16 + KP, J = (E + 31) / 32;
    __shared__ int cellbuf[4][E];
    __shared__ int pcellbuf[4][E];
    __shared__ int tokbuf[4][E];
    __shared__ int keybuf[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = int64_t(blockIdx.x) * 4 + warp;
    if (item >= items) return;
    const int img = int(uint32_t(item) / uint32_t(cs.c)), c = int(item) - img * cs.c;  // items < 2^31
    const int64_t img_tok = int64_t(img) * cs.n;
    const int32_t* nb = nbr_cl + item * cs.g;
    int32_t* out = qrec + item * R::WORDS;
    const int qlen = cs.len(c);
    // snapshot of the grid-wide radius max, read up front so its latency overlaps the gathers
    // (only used to skip atomics that cannot raise it; a stale value just costs an atomic)
    const int rmax_seen = lane == 0 ? *reinterpret_cast<volatile int*>(rmax) : 0;
    // equal-size clusters (N divisible by C, the lattice case): slot s is member s % base
    // of neighbour s / base, no per-slot walk over the groups
    const bool uniform = cs.rem == 0;
    int nk = 0;
    if (uniform) nk = cs.g * cs.base;
    else
        for (int g = 0; g < cs.g; ++g) nk += cs.len(nb[g]);
    TokAgg agg;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int e = lane + 32 * j;
        int tok = -1;
        if (e < 16) {
            if (e < qlen) tok = perm[img_tok + cs.off(c) + e];
        } else if (e < E && e - 16 < nk) {
            int s = e - 16;
            if (uniform) {
                const int g = s / cs.base;
                tok = perm[img_tok + __ldg(nb + g) * cs.base + (s - g * cs.base)];
            } else {
                for (int g = 0; g < cs.g; ++g) {
                    const int cl = nb[g], len = cs.len(cl);
                    if (s < len) {
                        tok = perm[img_tok + cs.off(cl) + s];
                        break;
                    }
                    s -= len;
                }
            }
        }
        int cell = 0, pcell = 0;
        if (tok >= 0) {
            const TokInfo t = make_tokinfo(reinterpret_cast<const float2*>(coords)[img_tok + tok], inv_patch);
            cell = tok_cell(t);
            pcell = tok_pcell(t);
            agg.far |= !pcell_ok(t);
            agg.add(t, e >= 16);
        }
        if (e < E) {
            tokbuf[warp][e] = tok;
            cellbuf[warp][e] = cell;
            pcellbuf[warp][e] = pcell;
        }
    }
    int radius = 0;
    const int cls = agg.cls(&radius);
    {   // one address for the whole grid: skip the atomic when it cannot raise the max
        const int rv = cls == 0 ? kRg : radius;
        if (lane == 0 && rv > rmax_seen) atomicMax(rmax, rv);
    }
    __syncwarp();
    if (cls == 1) {
        // Lattice-fast: reorder the key slots by (occurrence of the window
        // cell's residue mod 32, slot), so each 32-slot half holds distinct
        // residues where possible -- the backward's per-query-row table RMW
        // (lanes over key slots, bank = cell mod 32 + const) is then nearly
        // conflict-free.  Attention is invariant to the key order.
        const unsigned lt = (1u << lane) - 1u;
        const bool v0 = lane < nk, v1 = lane + 32 < nk;
        const int res0 = cellbuf[warp][16 + (lane < KP ? lane : 0)] & 31;
        const int res1 = KP > 32 ? cellbuf[warp][16 + (lane + 32 < KP ? lane + 32 : 0)] & 31 : 0;
        const unsigned m0 = __match_any_sync(0xffffffffu, v0 ? res0 : 64 + lane);
        const unsigned m1 = __match_any_sync(0xffffffffu, v1 ? res1 : 64 + lane);
        keybuf[warp][lane] = 0;  // per-residue count of the first half
        __syncwarp();
        if (v0) keybuf[warp][res0] = __popc(m0);
        __syncwarp();
        const int o0 = __popc(m0 & lt), o1 = (v1 ? keybuf[warp][res1] : 0) + __popc(m1 & lt);
        const int levels = __reduce_max_sync(0xffffffffu, max(v0 ? o0 : 0, v1 ? o1 : 0)) + 1;
        int npos[2] = {lane, lane + 32}, base = 0;
        for (int L = 0; L < levels; ++L) {
            const unsigned b0 = __ballot_sync(0xffffffffu, v0 && o0 == L);
            const unsigned b1 = __ballot_sync(0xffffffffu, v1 && o1 == L);
            if (v0 && o0 == L) npos[0] = base + __popc(b0 & lt);
            if (v1 && o1 == L) npos[1] = base + __popc(b0) + __popc(b1 & lt);
            base += __popc(b0) + __popc(b1);
        }
        int ntok[2], ncell[2], npcell[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int sl = lane + 32 * j;
            if (sl < nk) {
                ntok[j] = tokbuf[warp][16 + sl];
                ncell[j] = cellbuf[warp][16 + sl];
                npcell[j] = pcellbuf[warp][16 + sl];
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j)
            if (lane + 32 * j < nk) {
                tokbuf[warp][16 + npos[j]] = ntok[j];
                cellbuf[warp][16 + npos[j]] = ncell[j];
                pcellbuf[warp][16 + npos[j]] = npcell[j];
            }
        __syncwarp();
    }
    const int(*cb)[E] = cls == 2 ? pcellbuf : cellbuf;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int e = lane + 32 * j;
        if (e < E) {
            const bool valid = e < 16 ? e < qlen : e - 16 < nk;
            const int cell = valid ? cb[warp][e] : cb[warp][e < 16 ? 0 : 16];
            out[e < 16 ? R::QTOK + e : R::KTOK + e - 16] = tokbuf[warp][e];
            out[e < 16 ? R::QCELL + e : R::KCELL + e - 16] = cell;
        }
    }
    // duplicate key coordinates (exact packed cells; window cells alias beyond the window)
    const int ka = lane < nk ? pcellbuf[warp][16 + lane] : INT_MIN + lane;
    const int kb = lane + 32 < nk ? pcellbuf[warp][16 + lane + 32] : INT_MIN + 32 + lane;
    const bool anyfar = __any_sync(0xffffffffu, agg.far);
    const bool dup0 = anyfar || __any_sync(0xffffffffu, __popc(__match_any_sync(0xffffffffu, ka)) > 1);
    const bool dup1 = anyfar || __any_sync(0xffffffffu, __popc(__match_any_sync(0xffffffffu, kb)) > 1);
    if (lane < 8) {
        const int v = lane == kHNk ? nk : lane == kHQlen ? qlen : lane == kHFast ? cls
                    : lane == kHDup0 ? int(dup0) : lane == kHDup1 ? int(dup1)
                    : lane == kHImgTok ? int(img_tok) : lane == kHItem ? int(item) : 0;
        out[R::HDR + lane] = v;
    }
}

// Item lists, deterministic order: lattice-fast query clusters at
// list[0, n_fast), general ones at list[items, items + n_general), ascending.
// Pass 1 counts per 1024-item block, pass 2 offsets each block by the counts
// of the blocks before it and scatters.
__device__ __forceinline__ void block_flags_scan(bool fast, bool valid, int& pf, int& pg, int* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bf = __ballot_sync(0xffffffffu, fast), bg = __ballot_sync(0xffffffffu, valid && !fast);
    if (lane == 0) {
        wsum[warp] = __popc(bf);
        wsum[32 + warp] = __popc(bg);
    }
    __syncthreads();
    int af = 0, ag = 0;
    for (int w = 0; w < warp; ++w) {
        af += wsum[w];
        ag += wsum[32 + w];
    }
    const unsigned lt = (1u << lane) - 1u;
    pf = af + __popc(bf & lt);
    pg = ag + __popc(bg & lt);
}
__global__ void attn_item_count_kernel(const int32_t* __restrict__ qrec, int words, int hdr_fast, int items,
                                       int32_t* __restrict__ blk) {
    __shared__ int wsum[64];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < items;
    const bool fast = valid && qrec[size_t(i) * words + hdr_fast] == 1;
    int pf, pg;
    block_flags_scan(fast, valid, pf, pg, wsum);
    if (threadIdx.x == blockDim.x - 1) {
        blk[2 * blockIdx.x] = pf + int(fast);
        blk[2 * blockIdx.x + 1] = pg + int(valid && !fast);
    }
}
__global__ void attn_item_scatter_kernel(const int32_t* __restrict__ qrec, int words, int hdr_fast, int items,
                                         const int32_t* __restrict__ blk, int32_t* __restrict__ list,
                                         int32_t* __restrict__ count) {
    __shared__ int wsum[64];
    __shared__ int base[2];
    if (threadIdx.x < 2) {
        int b = 0;
        for (int k = 0; k < int(blockIdx.x); ++k) b += blk[2 * k + threadIdx.x];
        base[threadIdx.x] = b;
        if (blockIdx.x == gridDim.x - 1) count[threadIdx.x] = b + blk[2 * blockIdx.x + threadIdx.x];
    }
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < items;
    const bool fast = valid && qrec[size_t(i) * words + hdr_fast] == 1;
    int pf, pg;
    block_flags_scan(fast, valid, pf, pg, wsum);
    if (fast) list[base[0] + pf] = i;
    else if (valid) list[items + base[1] + pg] = i;
}

// Key-cluster records and reverse-pair records (one warp per key cluster c'):
// lanes 0..15 hold the key tokens, lanes 16..31 the query tokens of each pair
// (query clusters listing c' in their neighbourhood, CSR order).
__global__ void attn_krec_kernel(const float* __restrict__ coords, const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ rev_off, const int32_t* __restrict__ rev_cl,
                                 ClusterShape cs, int64_t items, float inv_patch,
                                 int32_t* __restrict__ krec, int32_t* __restrict__ prec) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = int64_t(blockIdx.x) * 4 + warp;
    if (item >= items) return;
    const int img = int(uint32_t(item) / uint32_t(cs.c)), ck = int(item) - img * cs.c;  // items < 2^31
    const int64_t img_tok = int64_t(img) * cs.n;
    const int64_t pairs = int64_t(cs.c) * cs.g;
    const int klen = cs.len(ck);
    const int rb = rev_off[int64_t(img) * (cs.c + 1) + ck], re = rev_off[int64_t(img) * (cs.c + 1) + ck + 1];
    int32_t* ko = krec + item * KRec::WORDS;
    // key side (lanes < 16)
    const bool kvalid = lane < klen;
    int ktok = -1;
    TokInfo kt{};
    if (kvalid) {
        ktok = perm[img_tok + cs.off(ck) + lane];
        kt = make_tokinfo(reinterpret_cast<const float2*>(coords)[img_tok + ktok], inv_patch);
    }
    const int kc = kvalid ? tok_cell(kt) : 0;
    const int kc0 = __shfl_sync(0xffffffffu, kc, 0);
    const int kpc = kvalid ? tok_pcell(kt) : 0;
    const int kpc0 = __shfl_sync(0xffffffffu, kpc, 0);
    const bool kfar = __any_sync(0xffffffffu, kvalid && !pcell_ok(kt));
    if (lane < 16) {
        ko[KRec::KTOK + lane] = ktok;
        ko[KRec::KCELL + lane] = kvalid ? kc : kc0;
        ko[KRec::KPCELL + lane] = kvalid ? kpc : kpc0;
    }
    if (lane < 8)
        ko[KRec::HDR + lane] = lane == 0 ? klen : lane == 1 ? rb : lane == 2 ? re
                             : lane == 3 ? int(int64_t(img) * pairs + rb) : lane == 4 ? int(img_tok) : 0;
    const Bbox kb = warp_bbox(kvalid, kt);
    for (int pr = rb; pr < re; ++pr) {
        const int qc = rev_cl[int64_t(img) * pairs + pr];
        const int qlen = cs.len(qc);
        const int qi = lane - 16;
        const bool qvalid = lane >= 16 && qi < qlen;
        int qtok = -1;
        TokInfo qt{};
        if (qvalid) {
            qtok = perm[img_tok + cs.off(qc) + qi];
            qt = make_tokinfo(reinterpret_cast<const float2*>(coords)[img_tok + qtok], inv_patch);
        }
        const Bbox qb = warp_bbox(qvalid, qt);
        const bool ph = warp_one_phase(kvalid || qvalid, kvalid ? kt : qt);
        const bool qfar = __any_sync(0xffffffffu, qvalid && !pcell_ok(qt));
        const int cls = !ph ? 0 : bbox_fits(qb, kb) ? 1 : (!kfar && !qfar && bbox_fits_r(qb, kb, kRg)) ? 2 : 0;
        const int qcell = qvalid ? (cls == 2 ? tok_pcell(qt) : tok_cell(qt)) : 0;
        const int qcell0 = __shfl_sync(0xffffffffu, qcell, 16);
        const int fast = cls;
        int32_t* po = prec + (int64_t(img) * pairs + pr) * PRec::WORDS;
        if (lane >= 16) {
            po[PRec::QTOK + qi] = qtok;
            po[PRec::QCELL + qi] = qvalid ? qcell : qcell0;
        }
        if (lane < 8) {
            const int v = lane == kPQlen ? qlen : lane == kPFast ? int(fast) : lane == kPFirst ? int(pr == rb)
                        : lane == kPLast ? int(pr == re - 1) : lane == kPItem ? int(item)
                        : lane == kPIdx ? int(int64_t(img) * pairs + pr)
                        : lane == kPQItem ? int(int64_t(img) * cs.c + qc)
                        : lane == kPImgTok ? int(img_tok) : 0;
            po[PRec::HDR + lane] = v;
        }
    }
}

// -------------------------------------------- BiasNet gradient finalize
// Per-CTA partials -> workspace gradient buffers, summed over CTAs in a fixed
// order (deterministic): window entries are added into the global table
// gradient (which also holds the tier-2 atomics), MLP and blank partials
// are written to their buffers.
// Block (entry chunk of 32, head): 8 warps split the CTA partials, fixed-order
// tree at the end (deterministic).
__global__ void attn_part_reduce_kernel(const float* __restrict__ part, int gx0, int gx1, int heads, int hd,
                                        int hidden, float* __restrict__ dtab_g, float* __restrict__ mlp_grad,
                                        float* __restrict__ blank_grad) {
    __shared__ float red[8][33];
    const int h = blockIdx.y;
    const int pw = part_width(hd);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + lane;
    float acc = 0.f;
    if (j < pw) {
        const float* p1 = part + size_t(heads) * gx0 * pw;
        auto at = [&](int x) {
            return x < gx0 ? part[(size_t(h) * gx0 + x) * pw + j] : p1[(size_t(h) * gx1 + x - gx0) * pw + j];
        };
        const int nx = gx0 + gx1;
        float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent chains, fixed order
        int x = warp;
        for (; x + 7 * 8 < nx; x += 64) {
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] += at(x + u * 8);
        }
        for (; x < nx; x += 8) a[0] += at(x);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += a[u];
    }
    red[warp][lane] = acc;
    __syncthreads();
    if (warp != 0 || j >= pw) return;
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red[w][lane];
    if (j < kWs2) {
        const int oy = j / kWs - kRs, ox = j % kWs - kRs;
        dtab_g[size_t(h) * kWg2 + (oy + kRg) * kWg + (ox + kRg)] += s;
    } else if (j < kWs2 + kMG) {
        const int u = j - kWs2;
        if (u <= 4 * hidden) mlp_grad[h * (4 * hidden + 1) + u] = s;
    } else {
        blank_grad[h * (2 * hd + 1) + (j - kWs2 - kMG)] = s;
    }
}

// dL/dtheta = sum over table entries of dT * dT/dtheta, accumulated (+=)
// into the caller's gradients.
// Sums the kTabReplicas copies of the table gradient into copy 0 (fixed order), used box only.
__global__ void dtab_replica_sum_kernel(float* __restrict__ dtab, int heads, const int32_t* __restrict__ rmax) {
    const int R = used_radius(rmax), side = 2 * R + 1, box = side * side;
    const size_t n = size_t(heads) * kWg2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < heads * box; i += gridDim.x * blockDim.x) {
        const int h = i / box, e = i - h * box;
        const int oy = e / side - R, ox = e - (e / side) * side - R;
        const size_t j = size_t(h) * kWg2 + (oy + kRg) * kWg + (ox + kRg);
        float v = dtab[j];
        for (int r = 1; r < kTabReplicas; ++r) v += dtab[r * n + j];
        dtab[j] = v;
    }
}

// dL/dtheta = sum over table entries of dT * dT/dtheta.  Pass 1: block b of head h
// folds the used-box entries b, b + nblk*256, ... into per-block partials
// {dw1x[H], dw1y[H], db1[H], dw2[H], db2}; pass 2 sums the block partials in a
// fixed order and adds them (+=) into the caller's gradients (deterministic).
__global__ void bias_grad_partial_kernel(const float* __restrict__ dtab, const float* __restrict__ w1,
                                         const float* __restrict__ b1, const float* __restrict__ w2, int hidden,
                                         const int32_t* __restrict__ rmax, float* __restrict__ fpart) {
    const int h = blockIdx.y;
    const float* dt = dtab + size_t(h) * kWg2;
    const int R = used_radius(rmax), side = 2 * R + 1, box = side * side;
    __shared__ float red[8][4 * kMaxHidden + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int stride = gridDim.x * blockDim.x, e0 = blockIdx.x * blockDim.x + threadIdx.x;
    auto entry = [&](int e, float& ox, float& oy) -> float {
        const int oyi = e / side, oxi = e - oyi * side;
        ox = float(oxi - R);
        oy = float(oyi - R);
        return dt[(oyi - R + kRg) * kWg + (oxi - R + kRg)];
    };
    {
        float sd = 0.f, ox, oy;
        for (int e = e0; e < box; e += stride) sd += entry(e, ox, oy);
        sd = warp_sum(sd);
        if (lane == 0) red[warp][4 * hidden] = sd;
    }
    for (int u = 0; u < hidden; ++u) {
        const float wx = w1[h * 2 * hidden + u], wy = w1[h * 2 * hidden + hidden + u];
        const float bb = b1[h * hidden + u], ww = w2[h * hidden + u];
        float gx = 0.f, gy = 0.f, gb = 0.f, gw = 0.f;
        for (int e = e0; e < box; e += stride) {
            float ox, oy;
            const float d = entry(e, ox, oy);
            if (d == 0.f) continue;
            const float t = tanhf(wx * ox + wy * oy + bb);
            const float dpre = d * ww * (1.f - t * t);
            gx = fmaf(dpre, ox, gx);
            gy = fmaf(dpre, oy, gy);
            gb += dpre;
            gw = fmaf(d, t, gw);
        }
        gx = warp_sum(gx);
        gy = warp_sum(gy);
        gb = warp_sum(gb);
        gw = warp_sum(gw);
        if (lane == 0) {
            red[warp][u] = gx;
            red[warp][hidden + u] = gy;
            red[warp][2 * hidden + u] = gb;
            red[warp][3 * hidden + u] = gw;
        }
    }
    __syncthreads();
    const int nv = 4 * hidden + 1;
    for (int j = threadIdx.x; j < nv; j += blockDim.x) {
        float s = 0.f;
        for (int w = 0; w < 8; ++w) s += red[w][j];
        fpart[(size_t(h) * gridDim.x + blockIdx.x) * nv + j] = s;
    }
}
__global__ void bias_grad_final_kernel(const float* __restrict__ fpart, int nblk, int hidden, float* dw1,
                                       float* db1, float* dw2, float* db2) {
    const int h = blockIdx.x, j = blockIdx.y;  // one warp per (head, parameter)
    const int nv = 4 * hidden + 1;
    float s = 0.f;
    for (int b = threadIdx.x; b < nblk; b += 32) s += fpart[(size_t(h) * nblk + b) * nv + j];
    s = warp_sum(s);
    if (threadIdx.x != 0) return;
    const int u = j % hidden, which = j / hidden;
    if (j == 4 * hidden) db2[h] += s;
    else if (which == 0) dw1[h * 2 * hidden + u] += s;
    else if (which == 1) dw1[h * 2 * hidden + hidden + u] += s;
    else if (which == 2) db1[h * hidden + u] += s;
    else dw2[h * hidden + u] += s;
}

// tier-3 partials and blank grads -> caller's gradient buffers (+=)
__global__ void attn_grad_epilogue_kernel(const float* __restrict__ mlp_grad,
                                          const float* __restrict__ blank_grad, int heads,
                                          int hidden, int hd, float* dw1, float* db1, float* dw2,
                                          float* db2, float* dbk, float* dbv, float* dblank) {
    const int h = blockIdx.x;
    const float* mg = mlp_grad + h * (4 * hidden + 1);
    const float* bg = blank_grad + h * (2 * hd + 1);
    for (int u = threadIdx.x; u < hidden; u += blockDim.x) {
        dw1[h * 2 * hidden + u] += mg[u];
        dw1[h * 2 * hidden + hidden + u] += mg[hidden + u];
        db1[h * hidden + u] += mg[2 * hidden + u];
        dw2[h * hidden + u] += mg[3 * hidden + u];
    }
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        dbk[h * hd + d] += bg[d];
        dbv[h * hd + d] += bg[hd + d];
    }
    if (threadIdx.x == 0) {
        db2[h] += mg[4 * hidden];
        dblank[h] += bg[2 * hd];
    }
}

template <int HD, int KP>
int launch_fwd(const AttnParams& p, cudaStream_t st);
template <int HD, int KP>
int launch_bwd_q(const AttnParams& p, cudaStream_t st, int* grid_x);
template <int HD>
int launch_bwd_kv(const AttnParams& p, cudaStream_t st);

// Key slots rounded up to a multiple of 16 (the blank sits at slot KP).
static int pick_kp(int64_t width) {
    if (width <= 16) return 16;
    if (width <= 32) return 32;
    if (width <= 48) return 48;
    if (width <= 64) return 64;
    return -1;
}

static int attn_check(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (!g || !a) return fail(AFFMAE_ECONFIG, "attention: null descriptor");
    if (g->n_clusters <= 0) return fail(AFFMAE_ECONFIG, "attention: geometry not derived (call affmae_cluster_geometry)");
    if (a->heads < 1 || a->head_dim < 1 || a->bias_hidden < 1 || !(a->patch > 0.0))
        return fail(AFFMAE_ECONFIG, "attention: heads, head_dim, bias_hidden, patch must be positive");
    if (a->head_dim != 16 && a->head_dim != 32 && a->head_dim != 64)
        return fail(AFFMAE_EUNSUPPORTED, "attention: head_dim must be 16, 32 or 64");
    if (g->max_size > 16)
        return fail(AFFMAE_EUNSUPPORTED, "attention: clusters larger than 16 tokens not compiled");
    if (pick_kp(g->width) < 0)
        return fail(AFFMAE_EUNSUPPORTED, "attention: neighbourhood width > 64 not compiled");
    if (a->bias_hidden > kMaxHidden) return fail(AFFMAE_EUNSUPPORTED, "attention: bias_hidden > 32");
    return AFFMAE_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Plan buffer (geometry only, reusable by every forward/backward on the same
// cluster index -- the reference's AttnOp freezes coords + NeighborIndex at
// construction, proj/src/attention.cpp:374-383): query-cluster records |
// item lists | [key records | pair records].  Its host descriptor
// (affmae_attn_plan) records what it was built for.
struct AttnWs {
    int32_t* qrec;
    int32_t* items;
    int32_t* item_count;
    int32_t* item_blk;
    int32_t* rmax;  // largest pair offset radius of the plan's items (bounds the BiasNet table box)
    int32_t* krec;
    int32_t* prec;
    float* tab_g;
    float* dtab_g;
    float2* lsd;
    float* part;
    float* mlp_grad;
    float* blank_grad;
    float* fpart;
    size_t plan_bytes, run_bytes;
};

struct Carver {
    uint8_t* p;
    size_t off = 0;
    uint8_t* take(size_t bytes) {
        uint8_t* r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    }
};

static void carve_plan(const affmae_cluster_geom* g, void* base, bool rev, AttnWs& w) {
    Carver c{static_cast<uint8_t*>(base)};
    const size_t items = size_t(g->batch) * g->n_clusters;
    const int kp = pick_kp(g->width);
    const size_t qwords = size_t(32 + 2 * kp + 8);
    w.qrec = reinterpret_cast<int32_t*>(c.take(items * qwords * 4));
    w.items = reinterpret_cast<int32_t*>(c.take(2 * items * 4));
    w.item_count = reinterpret_cast<int32_t*>(c.take(2 * 4));
    w.item_blk = reinterpret_cast<int32_t*>(c.take(2 * ((items + 1023) / 1024) * 4));
    w.rmax = reinterpret_cast<int32_t*>(c.take(16));
    if (rev) {
        w.krec = reinterpret_cast<int32_t*>(c.take(items * KRec::WORDS * 4));
        w.prec = reinterpret_cast<int32_t*>(c.take(items * g->groups_eff * PRec::WORDS * 4));
    }
    w.plan_bytes = c.off;
}

static void carve_run(const affmae_cluster_geom* g, const affmae_attn_desc* a, void* base, bool bwd,
                      AttnWs& w) {
    Carver c{static_cast<uint8_t*>(base)};
    w.tab_g = reinterpret_cast<float*>(c.take(size_t(a->heads) * kWg2 * 4));
    if (bwd) {
        w.dtab_g = reinterpret_cast<float*>(c.take(size_t(kTabReplicas) * a->heads * kWg2 * 4));
        w.lsd = reinterpret_cast<float2*>(c.take(size_t(g->batch) * g->n_clusters * a->heads * 16 * 8));
        w.part = reinterpret_cast<float*>(
            c.take(2 * size_t(kMaxCtasPerGroup) * a->heads * part_width(a->head_dim) * 4));  // [launch][h][CTA]
        w.mlp_grad = reinterpret_cast<float*>(c.take(size_t(a->heads) * (4 * a->bias_hidden + 1) * 4));
        w.blank_grad = reinterpret_cast<float*>(c.take(size_t(a->heads) * (2 * a->head_dim + 1) * 4));
        w.fpart = reinterpret_cast<float*>(
            c.take(size_t(a->heads) * kFinBlocks * (4 * a->bias_hidden + 1) * 4));
    }
    w.run_bytes = c.off;
}

// one-shot workspace = plan | run state
static AttnWs carve_ws(const affmae_cluster_geom* g, const affmae_attn_desc* a, void* base, bool bwd) {
    AttnWs w{};
    carve_plan(g, base, bwd, w);
    carve_run(g, a, base ? static_cast<uint8_t*>(base) + w.plan_bytes : nullptr, bwd, w);
    return w;
}

static void fill_common(AttnParams& p, const affmae_cluster_geom* g, const affmae_attn_desc* a,
                        const affmae_attn_inputs* in) {
    p = AttnParams{};
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
    p.cs = make_shape(*g);
    p.batch = int(g->batch);
    p.heads = a->heads;
    p.hidden = a->bias_hidden;
    p.inv_patch = float(1.0 / a->patch);
    p.scale = float(1.0 / sqrt(double(a->head_dim)));
    p.ldq = p.ldo = int64_t(a->heads) * a->head_dim;
}

static int check_inputs(const affmae_attn_inputs* in) {
    if (!in || !in->q || !in->k || !in->v || !in->blank_k || !in->blank_v || !in->coords ||
        !in->w1 || !in->b1 || !in->w2 || !in->b2 || !in->blank)
        return fail(AFFMAE_ECONFIG, "attention: null input pointer");
    return AFFMAE_OK;
}

// Geometry plan: query-cluster records, item lists (+ key / pair records).
static int build_plan(const affmae_cluster_geom* g, float inv_patch, const float* coords, const int32_t* perm,
                      const int32_t* nbr_cl, const int32_t* rev_off, const int32_t* rev_cl, const AttnWs& w,
                      cudaStream_t st) {
    const ClusterShape cs = make_shape(*g);
    const int64_t items = g->batch * g->n_clusters;
    const unsigned blocks = unsigned((items + 3) / 4);
    const int kp = pick_kp(g->width);
    // the key-side records (backward only) are independent of the query side:
    // build them concurrently on the forked side stream
    auto query_side = [&](cudaStream_t st) -> int {
        AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.rmax, 0, 16, st));
        switch (kp) {
#define AFFMAE_QREC(KP_)                                                                                 \
        case KP_:                                                                                            \
            attn_qrec_kernel<KP_><<<blocks, 128, 0, st>>>(coords, perm, nbr_cl, cs, items, inv_patch, w.qrec, \
                                                          w.rmax);                                           \
            break;
            AFFMAE_QREC(16)
            AFFMAE_QREC(32)
            AFFMAE_QREC(48)
            AFFMAE_QREC(64)
#undef AFFMAE_QREC
            default:
                return fail(AFFMAE_EUNSUPPORTED, "attention: width");
        }
        AFFMAE_LAUNCH_CHECK("attn_qrec_kernel");
        {
            const int words = 32 + 2 * kp + 8, hf = 32 + 2 * kp + kHFast;
            const unsigned nb = unsigned((items + 1023) / 1024);
            attn_item_count_kernel<<<nb, 1024, 0, st>>>(w.qrec, words, hf, int(items), w.item_blk);
            AFFMAE_LAUNCH_CHECK("attn_item_count_kernel");
            attn_item_scatter_kernel<<<nb, 1024, 0, st>>>(w.qrec, words, hf, int(items), w.item_blk, w.items,
                                                          w.item_count);
            AFFMAE_LAUNCH_CHECK("attn_item_scatter_kernel");
        }
        return AFFMAE_OK;
    };
    if (!rev_cl) return query_side(st);
    return launch_forked(
        st,
        [&](cudaStream_t s) {
            attn_krec_kernel<<<blocks, 128, 0, s>>>(coords, perm, rev_off, rev_cl, cs, items, inv_patch, w.krec,
                                                    w.prec);
            AFFMAE_LAUNCH_CHECK("attn_krec_kernel");
            return AFFMAE_OK;
        },
        query_side);
}

// per-call state: BiasNet offset table of the current weights; wires the plan in
static int prepare_run(AttnParams& p, const AttnWs& w, cudaStream_t st) {
    const int n = p.heads * kWg2;
    (void)n;
    bias_table_kernel<<<4 * kNumSMs, 256, 0, st>>>(p.w1, p.b1, p.w2, p.b2, p.heads, p.hidden, w.rmax, w.tab_g);
    AFFMAE_LAUNCH_CHECK("bias_table_kernel");
    p.tab_g = w.tab_g;
    p.qrec = w.qrec;
    p.items = w.items;
    p.item_count = w.item_count;
    p.krec = w.krec;
    p.prec = w.prec;
    return AFFMAE_OK;
}

static int dispatch_fwd(const AttnParams& p, int head_dim, int64_t width, cudaStream_t st) {
    const int kp = pick_kp(width);
#define AFFMAE_CASE(HD_, KP_) \
    if (head_dim == HD_ && kp == KP_) return launch_fwd<HD_, KP_>(p, st);
#define AFFMAE_CASE_HD(HD_) AFFMAE_CASE(HD_, 16) AFFMAE_CASE(HD_, 32) AFFMAE_CASE(HD_, 48) AFFMAE_CASE(HD_, 64)
    AFFMAE_CASE_HD(16)
    AFFMAE_CASE_HD(32)
    AFFMAE_CASE_HD(64)
#undef AFFMAE_CASE
    return fail(AFFMAE_EUNSUPPORTED, "attention: no compiled kernel variant");
}
static int dispatch_bwd_q(const AttnParams& p, int head_dim, int64_t width, cudaStream_t st, int* gx) {
    const int kp = pick_kp(width);
#define AFFMAE_CASE(HD_, KP_) \
    if (head_dim == HD_ && kp == KP_) return launch_bwd_q<HD_, KP_>(p, st, gx);
    AFFMAE_CASE_HD(16)
    AFFMAE_CASE_HD(32)
    AFFMAE_CASE_HD(64)
#undef AFFMAE_CASE
#undef AFFMAE_CASE_HD
    return fail(AFFMAE_EUNSUPPORTED, "attention: no compiled kernel variant");
}
static int dispatch_bwd_kv(const AttnParams& p, int head_dim, cudaStream_t st) {
    switch (head_dim) {
        case 16: return launch_bwd_kv<16>(p, st);
        case 32: return launch_bwd_kv<32>(p, st);
        case 64: return launch_bwd_kv<64>(p, st);
        default: return fail(AFFMAE_EUNSUPPORTED, "attention: no compiled kernel variant");
    }
}

size_t attn_fwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (attn_check(g, a)) return 0;
    const AttnWs w = carve_ws(g, a, nullptr, false);
    return w.plan_bytes + w.run_bytes;
}

size_t attn_bwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (attn_check(g, a)) return 0;
    const AttnWs w = carve_ws(g, a, nullptr, true);
    return w.plan_bytes + w.run_bytes;
}

size_t attn_plan_workspace(const affmae_cluster_geom* g, int with_reverse) {
    if (!g || g->n_clusters <= 0 || pick_kp(g->width) < 0) return 0;
    AttnWs w{};
    carve_plan(g, nullptr, with_reverse != 0, w);
    return w.plan_bytes;
}
size_t attn_fwd_planned_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (attn_check(g, a)) return 0;
    AttnWs w{};
    carve_run(g, a, nullptr, false, w);
    return w.run_bytes;
}
size_t attn_bwd_planned_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (attn_check(g, a)) return 0;
    AttnWs w{};
    carve_run(g, a, nullptr, true, w);
    return w.run_bytes;
}

int attn_plan_build(const affmae_cluster_geom* g, const affmae_attn_desc* a, const float* coords,
                    const affmae_cluster_index* idx, int with_reverse, affmae_attn_plan* plan, void* stream) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if (!coords || !idx || !idx->perm || !idx->nbr_cl || !plan || !plan->buf)
        return fail(AFFMAE_ECONFIG, "attn_plan_build: null pointer");
    if (with_reverse && (!idx->rev_off || !idx->rev_cl))
        return fail(AFFMAE_ECONFIG, "attn_plan_build: reverse CSR required for a backward plan");
    AttnWs w{};
    carve_plan(g, plan->buf, with_reverse != 0, w);
    if (plan->bytes < w.plan_bytes) return fail(AFFMAE_ECONFIG, "attn_plan_build: plan buffer too small");
    plan->batch = g->batch;
    plan->tokens = g->tokens;
    plan->n_clusters = g->n_clusters;
    plan->groups_eff = g->groups_eff;
    plan->width = g->width;
    plan->patch = a->patch;
    plan->has_reverse = with_reverse != 0;
    if (g->batch == 0) return AFFMAE_OK;
    return build_plan(g, float(1.0 / a->patch), coords, idx->perm, idx->nbr_cl,
                      with_reverse ? idx->rev_off : nullptr, with_reverse ? idx->rev_cl : nullptr, w,
                      as_stream(stream));
}

static int run_fwd(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
                   const AttnWs& w, affmae_bf16* out, float* lse, cudaStream_t st, int64_t ldq = 0) {
    AttnParams p;
    fill_common(p, g, a, in);
    if (ldq) p.ldq = ldq;
    p.out = reinterpret_cast<__nv_bfloat16*>(out);
    p.lse = lse;
    int rc = prepare_run(p, w, st);
    if (rc) return rc;
    return dispatch_fwd(p, a->head_dim, g->width, st);
}

static int run_bwd(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
                   const AttnWs& w, const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                   affmae_attn_grads* gr, cudaStream_t st, int64_t ldq = 0) {
    (void)out;
    AttnParams p;
    fill_common(p, g, a, in);
    if (ldq) p.ldq = ldq;
    p.lse = const_cast<float*>(lse);
    p.dout = reinterpret_cast<const __nv_bfloat16*>(dout);
    p.dq = reinterpret_cast<__nv_bfloat16*>(gr->dq);
    p.dk = reinterpret_cast<__nv_bfloat16*>(gr->dk);
    p.dv = reinterpret_cast<__nv_bfloat16*>(gr->dv);
    p.lsd = w.lsd;
    p.dtab_g = w.dtab_g;
    p.part = w.part;
    // BiasNet table (st) and the zeroed table-gradient replicas (side stream) are independent
    int rc = launch_forked(
        st,
        [&](cudaStream_t s) {
            dtab_zero_kernel<<<4 * kNumSMs, 256, 0, s>>>(w.dtab_g, a->heads, w.rmax);
            AFFMAE_LAUNCH_CHECK("dtab_zero_kernel");
            return AFFMAE_OK;
        },
        [&](cudaStream_t s) { return prepare_run(p, w, s); });
    if (rc) return rc;
    int gx[2] = {0, 0};
    if ((rc = dispatch_bwd_q(p, a->head_dim, g->width, st, gx))) return rc;
    // The parameter-gradient chain needs only the query side's partials: it runs on
    // the forked side stream while the key-side kernel (dK, dV) runs on `st`.
    auto param_grads = [&](cudaStream_t s) -> int {
        const int pw = part_width(a->head_dim);
        attn_part_reduce_kernel<<<dim3((pw + 31) / 32, a->heads), 256, 0, s>>>(
            w.part, gx[0], gx[1], a->heads, a->head_dim, a->bias_hidden, w.dtab_g, w.mlp_grad, w.blank_grad);
        AFFMAE_LAUNCH_CHECK("attn_part_reduce_kernel");
        dtab_replica_sum_kernel<<<2 * kNumSMs, 256, 0, s>>>(w.dtab_g, a->heads, w.rmax);
        AFFMAE_LAUNCH_CHECK("dtab_replica_sum_kernel");
        const int nblk = kFinBlocks;
        bias_grad_partial_kernel<<<dim3(nblk, a->heads), 256, 0, s>>>(w.dtab_g, in->w1, in->b1, in->w2,
                                                                     a->bias_hidden, w.rmax, w.fpart);
        AFFMAE_LAUNCH_CHECK("bias_grad_partial_kernel");
        bias_grad_final_kernel<<<dim3(a->heads, 4 * a->bias_hidden + 1), 32, 0, s>>>(
            w.fpart, nblk, a->bias_hidden, gr->dw1, gr->db1, gr->dw2, gr->db2);
        AFFMAE_LAUNCH_CHECK("bias_grad_final_kernel");
        attn_grad_epilogue_kernel<<<a->heads, 64, 0, s>>>(w.mlp_grad, w.blank_grad, a->heads, a->bias_hidden,
                                                          a->head_dim, gr->dw1, gr->db1, gr->dw2, gr->db2,
                                                          gr->dblank_k, gr->dblank_v, gr->dblank);
        AFFMAE_LAUNCH_CHECK("attn_grad_epilogue_kernel");
        return AFFMAE_OK;
    };
    return launch_forked(st, param_grads, [&](cudaStream_t s) { return dispatch_bwd_kv(p, a->head_dim, s); });
}

static int check_bwd_ptrs(const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                          const affmae_attn_grads* gr) {
    if (!out || !lse || !dout || !gr || !gr->dq || !gr->dk || !gr->dv || !gr->dblank_k || !gr->dblank_v ||
        !gr->dw1 || !gr->db1 || !gr->dw2 || !gr->db2 || !gr->dblank)
        return fail(AFFMAE_ECONFIG, "attn_bwd: null pointer");
    return AFFMAE_OK;
}

// A plan must have been built for this geometry / patch (and with the reverse CSR for a backward).
static int check_plan(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_plan* plan,
                      bool bwd, AttnWs& w) {
    if (!plan || !plan->buf) return fail(AFFMAE_ECONFIG, "attention: null plan");
    if (plan->batch != g->batch || plan->tokens != g->tokens || plan->n_clusters != g->n_clusters ||
        plan->groups_eff != g->groups_eff || plan->width != g->width || plan->patch != a->patch)
        return fail(AFFMAE_ECONFIG, "attention: plan was built for another geometry / patch");
    if (bwd && !plan->has_reverse)
        return fail(AFFMAE_ECONFIG, "attention: backward needs a plan built with the reverse CSR");
    carve_plan(g, plan->buf, plan->has_reverse != 0, w);
    return AFFMAE_OK;
}

int attn_fwd_planned(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
                     const affmae_attn_plan* plan, affmae_bf16* out, float* lse, void* workspace, size_t ws_bytes,
                     void* stream, int64_t ldq) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if ((rc = check_inputs(in))) return rc;
    if (!out || !lse) return fail(AFFMAE_ECONFIG, "attn_fwd: null pointer");
    cudaStream_t st = as_stream(stream);
    AttnWs w{};
    if ((rc = check_plan(g, a, plan, false, w))) return rc;
    carve_run(g, a, workspace, false, w);
    if (!workspace || ws_bytes < w.run_bytes) return fail(AFFMAE_ECONFIG, "attn_fwd: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    if (ldq && ldq < int64_t(a->heads) * a->head_dim) return fail(AFFMAE_ECONFIG, "attn_fwd: row stride too small");
    return run_fwd(g, a, in, w, out, lse, st, ldq);
}

int attn_bwd_planned(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
                     const affmae_attn_plan* plan, const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                     affmae_attn_grads* gr, void* workspace, size_t ws_bytes, void* stream, int64_t ldq) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if ((rc = check_inputs(in))) return rc;
    if ((rc = check_bwd_ptrs(out, lse, dout, gr))) return rc;
    cudaStream_t st = as_stream(stream);
    AttnWs w{};
    if ((rc = check_plan(g, a, plan, true, w))) return rc;
    carve_run(g, a, workspace, true, w);
    if (!workspace || ws_bytes < w.run_bytes) return fail(AFFMAE_ECONFIG, "attn_bwd: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    if (ldq && ldq < int64_t(a->heads) * a->head_dim) return fail(AFFMAE_ECONFIG, "attn_bwd: row stride too small");
    return run_bwd(g, a, in, w, out, lse, dout, gr, st, ldq);
}

int attn_fwd(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
             const int32_t* perm, const int32_t* nbr_cl, affmae_bf16* out, float* lse,
             void* workspace, size_t ws_bytes, void* stream) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if ((rc = check_inputs(in))) return rc;
    if (!perm || !nbr_cl || !out || !lse) return fail(AFFMAE_ECONFIG, "attn_fwd: null pointer");
    AttnWs w = carve_ws(g, a, workspace, false);
    if (!workspace || ws_bytes < w.plan_bytes + w.run_bytes)
        return fail(AFFMAE_ECONFIG, "attn_fwd: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    if ((rc = build_plan(g, float(1.0 / a->patch), in->coords, perm, nbr_cl, nullptr, nullptr, w, st))) return rc;
    return run_fwd(g, a, in, w, out, lse, st);
}

int attn_bwd(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
             const affmae_cluster_index* idx, const affmae_bf16* out, const float* lse,
             const affmae_bf16* dout, affmae_attn_grads* gr, void* workspace, size_t ws_bytes,
             void* stream) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if ((rc = check_inputs(in))) return rc;
    if (!idx || !idx->perm || !idx->nbr_cl || !idx->rev_off || !idx->rev_cl)
        return fail(AFFMAE_ECONFIG, "attn_bwd: null pointer");
    if ((rc = check_bwd_ptrs(out, lse, dout, gr))) return rc;
    AttnWs w = carve_ws(g, a, workspace, true);
    if (!workspace || ws_bytes < w.plan_bytes + w.run_bytes)
        return fail(AFFMAE_ECONFIG, "attn_bwd: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    if ((rc = build_plan(g, float(1.0 / a->patch), in->coords, idx->perm, idx->nbr_cl, idx->rev_off, idx->rev_cl,
                         w, st)))
        return rc;
    return run_bwd(g, a, in, w, out, lse, dout, gr, st);
}

}  // namespace affmae_b200
