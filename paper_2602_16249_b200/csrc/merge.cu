// Adaptive KNN token merge, batched (proj/src/merging.cpp):
//   retained_count / select_retained   merging.cpp:50-69   bit-exact
//   merge_plan                         merging.cpp:71-116  bit-exact
//   MergePoolOp forward / backward     merging.cpp:121-220 fp32 (values), exact indices
//
// select_retained: one stable radix sort of (image, descending-score key) with
// the token index as payload reproduces std::stable_sort's "score desc, ties
// to the lower index"; the first R of each image are flagged and compacted in
// index order (ascending output).
//
// merge_plan: the reference scans all R retained tokens for every dropped
// token (O(N R)).  Here the retained tokens of an image are bucketed in a
// uniform grid (~1 per cell) and each dropped token searches rings of cells
// around its own cell until the best (d^2, retained position) candidate is
// provably optimal: strictly closer than every unsearched cell, with a safety
// margin far above rounding.  d^2 is dx*dx + dy*dy in binary64 without FMA
// contraction, ties go to the lowest retained position, exactly the
// reference's first-minimum scan.  Pools collect (sqrt(d^2), j), are sorted
// by (dist, index) and truncated to k_m.
#include <algorithm>
#include <cmath>

#include "sort.cuh"

namespace affmae_b200 {

static unsigned blocks_of(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------- select_retained
__global__ void score_keys_kernel(const float* __restrict__ scores, int64_t batch, int64_t n,
                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * n) return;
    int64_t b = i / n;
    keys[i] = (uint64_t(b) << 32) | uint32_t(~float_order(scores[i]));  // larger score first
    vals[i] = uint32_t(i - b * n);
}

__global__ void keep_flags_kernel(const uint32_t* __restrict__ sorted_vals, int64_t batch, int64_t n,
                                  int64_t r, uint8_t* __restrict__ keep) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * n) return;
    int64_t b = i / n, pos = i - b * n;
    keep[b * n + sorted_vals[i]] = pos < r ? 1 : 0;
}

// one CTA per image: ascending compaction of the kept flags
__global__ void compact_kernel(const uint8_t* __restrict__ keep, int64_t n, int64_t r,
                               int32_t* __restrict__ out) {
    __shared__ int32_t part[1024];
    const int t = threadIdx.x, nt = blockDim.x;
    const uint8_t* k = keep + int64_t(blockIdx.x) * n;
    const int64_t per = (n + nt - 1) / nt, b = t * per, e = (b + per < n) ? b + per : n;
    int32_t s = 0;
    for (int64_t i = b; i < e; ++i) s += k[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        int32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t pos = part[t] - s;
    int32_t* o = out + int64_t(blockIdx.x) * r;
    for (int64_t i = b; i < e; ++i)
        if (k[i]) o[pos++] = int32_t(i);
}

// ------------------------------------------------- select_retained by radix select
// One CTA per image (n <= kSegSortMax).  Keys w = ~float_order(score): the
// retained set is the r smallest keys, ties -> lower index, i.e. the first r of
// the stable ascending order (std::stable_sort by score desc,
// proj/src/merging.cpp:56-69).  Four MSB-first 8-bit histogram passes find the
// r-th key T and how many keys equal to T are taken; a stable compaction then
// writes the selected indices in ascending order.
constexpr int kSelWarps = 32;
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wsum, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t x = lane < kSelWarps ? wsum[lane] : 0u, xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, d);
            if (lane >= d) xi += y;
        }
        wsum[lane] = xi - x;
        if (lane == 31) wsum[32] = xi;
    }
    __syncthreads();
    const uint32_t r = wsum[warp] + inc - v;
    total = wsum[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kSelWarps * 32) select_topk_kernel(const float* __restrict__ scores, int64_t n,
                                                                     int64_t r, int32_t* __restrict__ out) {
    extern __shared__ uint32_t sw[];  // n keys
    __shared__ uint32_t hist[kSelWarps][257];
    __shared__ uint32_t wsum[33];
    __shared__ uint32_t bc[2];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int N = int(n);
    const float* s = scores + int64_t(blockIdx.x) * n;
    for (int i0 = t; i0 < N; i0 += 8 * kSelWarps * 32) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * kSelWarps * 32;
            v[u] = i < N ? __ldg(s + i) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * kSelWarps * 32;
            if (i < N) sw[i] = ~float_order(v[u]);
        }
    }
    const int per = ((((N + 31) / 32) + kSelWarps - 1) / kSelWarps) * 32;
    const int w0 = warp * per, w1 = min(w0 + per, N);
    uint32_t prefix = 0, mask = 0, need = uint32_t(r);
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = t; i < kSelWarps * 257; i += blockDim.x) (&hist[0][0])[i] = 0;
        __syncthreads();
        for (int b = w0; b < w1; b += 32) {
            const int i = b + lane;
            int d = 256;
            if (i < w1) {
                const uint32_t w = sw[i];
                if ((w & mask) == prefix) d = int((w >> shift) & 0xFF);
            }
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256 && __popc(peers & lt) == 0) hist[warp][d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        if (warp == 0) {  // digit where the cumulative count reaches `need`
            uint32_t c[8], run = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint32_t x = 0;
                for (int w = 0; w < kSelWarps; ++w) x += hist[w][lane * 8 + j];
                c[j] = x;
                run += x;
            }
            uint32_t inc = run;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += y;
            }
            const uint32_t before = inc - run;
            const unsigned hit = __ballot_sync(0xffffffffu, inc >= need && before < need);
            if (lane == __ffs(hit) - 1) {
                uint32_t acc = before;
                int dsel = 7;
                for (int j = 0; j < 8; ++j) {
                    if (acc + c[j] >= need) {
                        dsel = j;
                        break;
                    }
                    acc += c[j];
                }
                bc[0] = uint32_t(lane * 8 + dsel);
                bc[1] = acc;
            }
        }
        __syncthreads();
        prefix |= bc[0] << shift;
        mask |= 0xFFu << shift;
        need -= bc[1];
        __syncthreads();
    }
    // stable compaction: w < T, or w == T among the first `need` equal keys (index order)
    const uint32_t T = prefix;
    uint32_t eq = 0;
    for (int b = w0; b < w1; b += 32) {
        const int i = b + lane;
        eq += __popc(__ballot_sync(0xffffffffu, i < w1 && sw[i] == T));
    }
    uint32_t tot;
    uint32_t eq_before = block_excl_scan(lane == 0 ? eq : 0u, wsum, tot);
    eq_before = __shfl_sync(0xffffffffu, eq_before, 0);
    uint32_t sel = 0, eqr = eq_before;
    for (int b = w0; b < w1; b += 32) {
        const int i = b + lane;
        const uint32_t w = i < w1 ? sw[i] : 0xffffffffu;
        const unsigned be = __ballot_sync(0xffffffffu, i < w1 && w == T);
        const bool take = i < w1 && (w < T || (w == T && eqr + __popc(be & lt) < need));
        sel += __popc(__ballot_sync(0xffffffffu, take));
        eqr += __popc(be);
    }
    uint32_t sel_before = block_excl_scan(lane == 0 ? sel : 0u, wsum, tot);
    sel_before = __shfl_sync(0xffffffffu, sel_before, 0);
    int32_t* o = out + int64_t(blockIdx.x) * r;
    uint32_t pos = sel_before;
    eqr = eq_before;
    for (int b = w0; b < w1; b += 32) {
        const int i = b + lane;
        const uint32_t w = i < w1 ? sw[i] : 0xffffffffu;
        const unsigned be = __ballot_sync(0xffffffffu, i < w1 && w == T);
        const bool take = i < w1 && (w < T || (w == T && eqr + __popc(be & lt) < need));
        const unsigned bt = __ballot_sync(0xffffffffu, take);
        if (take) o[pos + __popc(bt & lt)] = i;
        pos += __popc(bt);
        eqr += __popc(be);
    }
}

// --------------------------------------------------------------- merge_plan
struct GridPrm {
    double x0, y0, w;  // origin and cell width
};

// per image bounding box -> grid of G x G cells (one CTA per image)
__global__ void grid_prm_kernel(const float* __restrict__ coords, int64_t n, int g,
                                GridPrm* __restrict__ prm) {
    __shared__ float red[4][32];
    const float2* xy = reinterpret_cast<const float2*>(coords) + int64_t(blockIdx.x) * n;
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        float2 v = xy[i];
        mnx = fminf(mnx, v.x);
        mny = fminf(mny, v.y);
        mxx = fmaxf(mxx, v.x);
        mxy = fmaxf(mxy, v.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        red[0][warp] = mnx;
        red[1][warp] = mny;
        red[2][warp] = mxx;
        red[3][warp] = mxy;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) {
            mnx = fminf(mnx, red[0][w]);
            mny = fminf(mny, red[1][w]);
            mxx = fmaxf(mxx, red[2][w]);
            mxy = fmaxf(mxy, red[3][w]);
        }
        double ext = fmax(double(mxx) - double(mnx), double(mxy) - double(mny));
        GridPrm p;
        p.x0 = mnx;
        p.y0 = mny;
        p.w = ext > 0.0 ? ext / g * (1.0 + 1e-9) : 1.0;
        prm[blockIdx.x] = p;
    }
}

__device__ __forceinline__ int cell_of(double v, double v0, double w, int g) {
    int c = int(floor((v - v0) / w));
    return c < 0 ? 0 : (c >= g ? g - 1 : c);
}

__global__ void mark_retained_kernel(const int32_t* __restrict__ retained, int64_t batch, int64_t n,
                                     int64_t r, int32_t* __restrict__ ret_pos) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * r) return;
    int64_t b = i / r;
    ret_pos[b * n + retained[i]] = int32_t(i - b * r);
}

__global__ void cell_count_kernel(const float* __restrict__ coords, const int32_t* __restrict__ retained,
                                  int64_t batch, int64_t n, int64_t r, int g,
                                  const GridPrm* __restrict__ prm, int32_t* __restrict__ cnt) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * r) return;
    int64_t b = i / r;
    const GridPrm p = prm[b];
    float2 v = reinterpret_cast<const float2*>(coords)[b * n + retained[i]];
    int cx = cell_of(v.x, p.x0, p.w, g), cy = cell_of(v.y, p.y0, p.w, g);
    atomicAdd(cnt + b * (int64_t(g) * g + 1) + cy * g + cx, 1);
}

// one CTA per segment: exclusive scan in place over len entries
__global__ void seg_scan_kernel(int32_t* __restrict__ cnt, int64_t len) {
    __shared__ int32_t part[1024];
    int32_t* c = cnt + int64_t(blockIdx.x) * len;
    const int t = threadIdx.x, nt = blockDim.x;
    const int64_t per = (len + nt - 1) / nt, b = t * per, e = (b + per < len) ? b + per : len;
    int32_t s = 0;
    for (int64_t i = b; i < e; ++i) s += c[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        int32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - s;
    for (int64_t i = b; i < e; ++i) {
        int32_t v = c[i];
        c[i] = run;
        run += v;
    }
}

__global__ void cell_fill_kernel(const float* __restrict__ coords, const int32_t* __restrict__ retained,
                                 int64_t batch, int64_t n, int64_t r, int g,
                                 const GridPrm* __restrict__ prm, const int32_t* __restrict__ off,
                                 int32_t* __restrict__ cursor, int32_t* __restrict__ items,
                                 float2* __restrict__ item_xy) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * r) return;
    int64_t b = i / r;
    const GridPrm p = prm[b];
    float2 v = reinterpret_cast<const float2*>(coords)[b * n + retained[i]];
    int cx = cell_of(v.x, p.x0, p.w, g), cy = cell_of(v.y, p.y0, p.w, g);
    int64_t cell = b * (int64_t(g) * g + 1) + cy * g + cx;
    int slot = atomicAdd(cursor + cell, 1);
    items[b * r + off[cell] + slot] = int32_t(i - b * r);
    item_xy[b * r + off[cell] + slot] = v;  // candidate coordinates beside the index: one load per candidate
}

__device__ __forceinline__ bool better(double d, int ri, double bd, int bri) {
    return bri < 0 || d < bd || (d == bd && ri < bri);
}
// fp32 pre-filter of the binary64 distance (index.cu knn_d2f): the fp32 squared distance is
// within a relative 2^-21 of the binary64 one, so a candidate whose fp32 value exceeds
// (1 + 2^-17) * best cannot win (nor tie) and skips the FP64 arithmetic.
__device__ __forceinline__ float d2_f32(float2 p, float2 q) {
    const float dx = __fsub_rn(p.x, q.x), dy = __fsub_rn(p.y, q.y);
    return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

// exact nearest retained token of every dropped token (first-minimum rule)
__global__ void assign_kernel(const float* __restrict__ coords, const int32_t* __restrict__ retained,
                              const int32_t* __restrict__ ret_pos, int64_t batch, int64_t n, int64_t r,
                              int g, const GridPrm* __restrict__ prm, const int32_t* __restrict__ off,
                              const int32_t* __restrict__ items, const float2* __restrict__ item_xy,
                              int32_t* __restrict__ target,
                              int32_t* __restrict__ best_of, double* __restrict__ d2_of,
                              int32_t* __restrict__ pool_cnt_all) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * n) return;
    int64_t b = i / n;
    if (ret_pos[i] >= 0) {
        target[i] = -1;
        best_of[i] = -1;
        return;
    }
    const GridPrm p = prm[b];
    const float2* xy = reinterpret_cast<const float2*>(coords) + b * n;
    const int32_t* ret = retained + b * r;
    const int32_t* co = off + b * (int64_t(g) * g + 1);
    const int32_t* it = items + b * r;
    const float2* ixy = item_xy + b * r;
    const float2 q = xy[i - b * n];
    const double qx = q.x, qy = q.y;
    const int qcx = cell_of(qx, p.x0, p.w, g), qcy = cell_of(qy, p.y0, p.w, g);
    double bd = 0.0;
    int bri = -1;
    float thr = INFINITY;
    for (int ring = 0; ring <= g; ++ring) {
        const int x0 = qcx - ring, x1 = qcx + ring, y0 = qcy - ring, y1 = qcy + ring;
        auto visit = [&](int cx, int cy) {
            const int cell = cy * g + cx;
            for (int t = co[cell]; t < co[cell + 1]; ++t) {
                const float2 v = ixy[t];
                if (d2_f32(v, q) > thr) continue;
                const int ri = it[t];
                const double dx = __dsub_rn(double(v.x), qx), dy = __dsub_rn(double(v.y), qy);
                const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                if (better(d2, ri, bd, bri)) {
                    bd = d2;
                    bri = ri;
                    thr = bd < 1e37 ? __double2float_ru(bd * (1.0 + 0x1p-17)) : INFINITY;
                }
            }
        };
        // perimeter of the (2 ring + 1)^2 block, clipped to the grid
        for (int cy = max(y0, 0); cy <= min(y1, g - 1); ++cy) {
            if (cy == y0 || cy == y1) {
                for (int cx = max(x0, 0); cx <= min(x1, g - 1); ++cx) visit(cx, cy);
            } else {
                if (x0 >= 0) visit(x0, cy);
                if (x1 <= g - 1 && x1 != x0) visit(x1, cy);
            }
        }
        if (bri >= 0) {
            // distance from q to the outside of the searched (2 ring + 1)^2 block
            double lb = INFINITY;
            if (x0 > 0) lb = fmin(lb, qx - (p.x0 + x0 * p.w));
            if (x1 < g - 1) lb = fmin(lb, p.x0 + (x1 + 1) * p.w - qx);
            if (y0 > 0) lb = fmin(lb, qy - (p.y0 + y0 * p.w));
            if (y1 < g - 1) lb = fmin(lb, p.y0 + (y1 + 1) * p.w - qy);
            if (lb == INFINITY) break;  // whole grid searched
            lb -= 1e-6 * p.w;
            if (lb > 0.0 && bd < lb * lb) break;
        }
    }
    target[i] = ret[bri];
    best_of[i] = bri;
    d2_of[i] = bd;
    atomicAdd(pool_cnt_all + b * (r + 1) + bri, 1);
}

__global__ void pool_fill_kernel(const int32_t* __restrict__ best_of, const double* __restrict__ d2_of,
                                 int64_t batch, int64_t n, int64_t r, const int32_t* __restrict__ off,
                                 int32_t* __restrict__ cursor, double* __restrict__ ldist,
                                 int32_t* __restrict__ lidx) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * n) return;
    int ri = best_of[i];
    if (ri < 0) return;
    int64_t b = i / n;
    int64_t seg = b * (r + 1) + ri;
    int slot = atomicAdd(cursor + seg, 1);
    int64_t pos = b * n + off[seg] + slot;
    ldist[pos] = __dsqrt_rn(d2_of[i]);
    lidx[pos] = int32_t(i - b * n);
}

// per retained token (one warp): the k_m smallest (dist, index) pairs of its candidate list,
// ascending (the reference sorts the whole pool and truncates, merging.cpp:102-114; only the
// kept prefix is observable).  Lanes stride over the list keeping a register-sorted top-K,
// then K rounds of a warp-wide lexicographic minimum.  O(list) per pool: with spatially
// clustered retained tokens one pool can collect thousands of candidates.
constexpr int kPoolK = 16;
__device__ __forceinline__ bool pair_less(double da, int ja, double db, int jb) {
    return da < db || (da == db && ja < jb);
}
// warp-cooperative top-k_m of one long candidate list (the list of pool i)
__device__ void pool_topk_warp(int64_t i, int lane, const int32_t* __restrict__ off, int64_t n, int64_t r, int k_m,
                               const double* __restrict__ ldist, const int32_t* __restrict__ lidx,
                               int32_t* __restrict__ pool_idx, double* __restrict__ pool_dist,
                               int32_t* __restrict__ pool_cnt, int32_t* __restrict__ row_of,
                               const int32_t* __restrict__ retained) {
    const int64_t b = i / r;
    const int ri = int(i - b * r);
    const int32_t* o = off + b * (r + 1);
    const double* ld = ldist + b * n;
    const int32_t* li = lidx + b * n;
    const int s = o[ri], e = o[ri + 1];
    double d[kPoolK];
    int j[kPoolK];
#pragma unroll
    for (int t = 0; t < kPoolK; ++t) {
        d[t] = INFINITY;
        j[t] = INT_MAX;
    }
    for (int x = s + lane; x < e; x += 32) {
        double dv = ld[x];
        int jv = li[x];
        if (!pair_less(dv, jv, d[kPoolK - 1], j[kPoolK - 1])) continue;
#pragma unroll
        for (int t = 0; t < kPoolK; ++t) {  // insertion into the sorted list
            if (pair_less(dv, jv, d[t], j[t])) {
                const double td = d[t];
                const int tj = j[t];
                d[t] = dv;
                j[t] = jv;
                dv = td;
                jv = tj;
            }
        }
    }
    const int keep = min(e - s, k_m);
    double thr_d = -INFINITY;
    int thr_j = -1;
    int head = 0;
    for (int t = 0; t < keep; ++t) {
        double cd = INFINITY;
        int cj = INT_MAX;
#pragma unroll
        for (int q = 0; q < kPoolK; ++q)
            if (q == head) {
                cd = d[q];
                cj = j[q];
            }
        double md = cd;
        int mj = cj;
#pragma unroll
        for (int ofs = 16; ofs > 0; ofs >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, md, ofs);
            const int oj = __shfl_xor_sync(0xffffffffu, mj, ofs);
            if (pair_less(od, oj, md, mj)) {
                md = od;
                mj = oj;
            }
        }
        if (cd == md && cj == mj) ++head;  // pairs are unique: exactly one lane owns the minimum
        if (lane == 0) {
            pool_idx[i * k_m + t] = mj;
            pool_dist[i * k_m + t] = md;
        }
        thr_d = md;
        thr_j = mj;
    }
    if (lane == 0) {
        for (int t = keep; t < k_m; ++t) {
            pool_idx[i * k_m + t] = -1;
            pool_dist[i * k_m + t] = 0.0;
        }
        pool_cnt[i] = keep;
        row_of[b * n + retained[i]] = ri;
    }
    for (int x = s + lane; x < e; x += 32)
        row_of[b * n + li[x]] = pair_less(thr_d, thr_j, ld[x], li[x]) ? -1 : ri;
}

// A warp per 32 pools: each lane sorts its own (short) candidate list by insertion, the lists
// longer than 32 are then taken one at a time by the whole warp.  Balanced pools (random
// scores: ~1.5 candidates) stay one-thread work; spatially clustered retained tokens (the
// model's learned scores) can give one pool thousands of candidates.
constexpr int kPoolShort = 32;
__global__ void __launch_bounds__(256) pool_topk_kernel(const int32_t* __restrict__ off, int64_t batch, int64_t n,
                                                        int64_t r, int k_m, double* __restrict__ ldist,
                                                        int32_t* __restrict__ lidx, int32_t* __restrict__ pool_idx,
                                                        double* __restrict__ pool_dist, int32_t* __restrict__ pool_cnt,
                                                        int32_t* __restrict__ row_of,
                                                        const int32_t* __restrict__ retained) {
    const int lane = threadIdx.x & 31;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool ok = i < batch * r;
    bool is_long = false;
    if (ok) {
        const int64_t b = i / r;
        const int ri = int(i - b * r);
        const int32_t* o = off + b * (r + 1);
        double* ld = ldist + b * n;
        int32_t* li = lidx + b * n;
        const int s = o[ri], e = o[ri + 1];
        is_long = e - s > kPoolShort;
        if (!is_long) {
            for (int x = s + 1; x < e; ++x) {
                const double dv = ld[x];
                const int iv = li[x];
                int y = x;
                while (y > s && (ld[y - 1] > dv || (ld[y - 1] == dv && li[y - 1] > iv))) {
                    ld[y] = ld[y - 1];
                    li[y] = li[y - 1];
                    --y;
                }
                ld[y] = dv;
                li[y] = iv;
            }
            const int keep = min(e - s, k_m);
            pool_cnt[i] = keep;
            for (int t = 0; t < k_m; ++t) {
                pool_idx[i * k_m + t] = t < keep ? li[s + t] : -1;
                pool_dist[i * k_m + t] = t < keep ? ld[s + t] : 0.0;
            }
            row_of[b * n + retained[i]] = ri;
            for (int t = 0; t < e - s; ++t) row_of[b * n + li[s + t]] = t < keep ? ri : -1;
        }
    }
    unsigned todo = __ballot_sync(0xffffffffu, is_long);
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t i2 = __shfl_sync(0xffffffffu, i, src);
        pool_topk_warp(i2, lane, off, n, r, k_m, ldist, lidx, pool_idx, pool_dist, pool_cnt, row_of, retained);
    }
}

// ---------------------------------------------------- pool forward/backward
// pool weights of one retained row: softmax(-p * dist) over its pool
__device__ __forceinline__ int pool_weights(const double* dist, int cnt, float p, float* w) {
    float m = -INFINITY;
    for (int t = 0; t < cnt; ++t) m = fmaxf(m, -p * float(dist[t]));
    float l = 0.f;
    for (int t = 0; t < cnt; ++t) {
        w[t] = __expf(-p * float(dist[t]) - m);
        l += w[t];
    }
    const float il = 1.f / l;
    for (int t = 0; t < cnt; ++t) w[t] *= il;
    return cnt;
}

constexpr int kMaxKm = 16;

// one warp per retained row: out = [f_r ; sum_t w_t s_j f_j]   (merging.cpp:121-149)
__global__ void pool_fwd_kernel(const __nv_bfloat16* __restrict__ feats, const float* __restrict__ scores,
                                const float* __restrict__ p_merge, const int32_t* __restrict__ retained,
                                const int32_t* __restrict__ pool_idx, const double* __restrict__ pool_dist,
                                const int32_t* __restrict__ pool_cnt, int64_t batch, int64_t n, int64_t r,
                                int dim, int k_m, __nv_bfloat16* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= batch * r) return;
    int64_t b = row / r;
    const float p = *p_merge;
    const int cnt = pool_cnt[row];
    float w[kMaxKm];
    pool_weights(pool_dist + row * k_m, cnt, p, w);
    const __nv_bfloat16* fb = feats + b * n * dim;
    const int32_t* pi = pool_idx + row * k_m;
    __nv_bfloat16* o = out + row * 2 * dim;
    const __nv_bfloat16* fr = fb + int64_t(retained[row]) * dim;
    for (int c = lane * 2; c < dim; c += 64) {
        *reinterpret_cast<__nv_bfloat162*>(o + c) = *reinterpret_cast<const __nv_bfloat162*>(fr + c);
        float a0 = 0.f, a1 = 0.f;
        for (int t = 0; t < cnt; ++t) {
            const int j = pi[t];
            const float g = w[t] * scores[b * n + j];
            float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(fb + int64_t(j) * dim + c));
            a0 = fmaf(g, f.x, a0);
            a1 = fmaf(g, f.y, a1);
        }
        *reinterpret_cast<__nv_bfloat162*>(o + dim + c) = __floats2bfloat162_rn(a0, a1);
    }
}

// one warp per retained row (MergePoolOp::backward, merging.cpp:169-219):
//   df[r] = g_left;  df[j] = g_right w_t s_j;  ds[j] = w_t <g_right, f_j>;
//   dp += sum_t w_t (dw_t - sum w dw) (-dist_t),  dw_t = s_j <g_right, f_j>
__global__ void pool_bwd_kernel(const __nv_bfloat16* __restrict__ feats, const float* __restrict__ scores,
                                const float* __restrict__ p_merge, const int32_t* __restrict__ retained,
                                const int32_t* __restrict__ pool_idx, const double* __restrict__ pool_dist,
                                const int32_t* __restrict__ pool_cnt, int64_t batch, int64_t n, int64_t r,
                                int dim, int k_m, const __nv_bfloat16* __restrict__ dout,
                                __nv_bfloat16* __restrict__ dfeats, float* __restrict__ dscores,
                                float* __restrict__ dp_part) {
    const int lane = threadIdx.x & 31;
    int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    float dp = 0.f;
    if (row < batch * r) {
        int64_t b = row / r;
        const float p = *p_merge;
        const int cnt = pool_cnt[row];
        const double* dist = pool_dist + row * k_m;
        float w[kMaxKm];
        pool_weights(dist, cnt, p, w);
        const __nv_bfloat16* fb = feats + b * n * dim;
        const __nv_bfloat16* g = dout + row * 2 * dim;
        const int32_t* pi = pool_idx + row * k_m;
        __nv_bfloat16* dfb = dfeats + b * n * dim;
        const int64_t rtok = retained[row];
        for (int c = lane * 2; c < dim; c += 64)
            *reinterpret_cast<__nv_bfloat162*>(dfb + rtok * dim + c) =
                *reinterpret_cast<const __nv_bfloat162*>(g + c);
        if (lane == 0) dscores[b * n + rtok] = 0.f;
        float dw[kMaxKm];
        float wdot = 0.f;
        for (int t = 0; t < cnt; ++t) {
            const int64_t j = pi[t];
            const float sj = scores[b * n + j];
            float dot = 0.f;
            for (int c = lane * 2; c < dim; c += 64) {
                float2 go = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(g + dim + c));
                float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(fb + j * dim + c));
                dot = fmaf(go.x, f.x, fmaf(go.y, f.y, dot));
                const float k = w[t] * sj;
                *reinterpret_cast<__nv_bfloat162*>(dfb + j * dim + c) = __floats2bfloat162_rn(go.x * k, go.y * k);
            }
            dot = warp_sum(dot);
            if (lane == 0) dscores[b * n + j] = w[t] * dot;
            dw[t] = sj * dot;
            wdot = fmaf(w[t], dw[t], wdot);
        }
        for (int t = 0; t < cnt; ++t) dp = fmaf(w[t] * (dw[t] - wdot), -float(dist[t]), dp);
    }
    // block partial of dp (deterministic order inside the block)
    __shared__ float red[32];
    const int warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = dp;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
        dp_part[blockIdx.x] = s;
    }
}

// tokens that feed no output row (truncated pool members) get zero gradient
__global__ void pool_bwd_zero_kernel(const int32_t* __restrict__ row_of, int64_t total, int dim,
                                     __nv_bfloat16* __restrict__ dfeats, float* __restrict__ dscores) {
    const int lane = threadIdx.x & 31;
    int64_t tok = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (tok >= total || row_of[tok] >= 0) return;
    for (int c = lane * 2; c < dim; c += 64)
        *reinterpret_cast<__nv_bfloat162*>(dfeats + tok * dim + c) = __floats2bfloat162_rn(0.f, 0.f);
    if (lane == 0) dscores[tok] = 0.f;
}

// dp += sum of block partials (one CTA, fixed reduction order)
__global__ void dp_reduce_kernel(const float* __restrict__ part, int nparts, float* __restrict__ dp) {
    __shared__ float red[32];
    float s = 0.f;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        *dp += t;
    }
}

// ------------------------------------------- vectorised pool kernels (dim % 8 == 0)
// A row of D bf16 is CPR = D/8 16-byte chunks (MergePoolOp, merging.cpp:121-220).
__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float (&f)[8]) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}

// tokens that feed no output row (truncated pool members): zero gradient (thread per token)
template <int CPR>
__global__ void pool_bwd_zero_vec_kernel(const int32_t* __restrict__ row_of, int64_t total,
                                        __nv_bfloat16* __restrict__ dfeats, float* __restrict__ dscores) {
    const int64_t tok = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tok >= total || row_of[tok] >= 0) return;
    uint4* d = reinterpret_cast<uint4*>(dfeats) + tok * CPR;
    for (int c = 0; c < CPR; ++c) d[c] = make_uint4(0, 0, 0, 0);
    dscores[tok] = 0.f;
}

// ------------------------------------------- staged pool kernels (persistent)
// Each warp walks rounds of RPW retained rows (LPR lanes per row, CPL 16-byte
// chunks per lane).  Round i+1's member rows (and the pool metadata: member
// ids, softmax weights, distances, member scores) are gathered by cp.async
// into a per-warp two-stage shared-memory ring while round i computes, and the
// pool indices of round i+2 load into registers one round earlier still -- so
// the in-flight data lives in shared memory, not in registers, and every warp
// keeps two rounds of gathers in flight.  Same arithmetic, same order as the
// v2 kernels (the results are bit-identical).
template <int CPR>
struct PoolGeo {
    static constexpr int LPR = CPR < 16 ? CPR : 16;  // lanes per row
    static constexpr int RPW = 32 / LPR;             // rows per warp round
    static constexpr int CPL = CPR / LPR;            // chunks per lane
    static constexpr int WARPS = CPR <= 16 ? 8 : CPR == 32 ? 4 : 2;
};
template <int KMAX>
struct PoolMeta {  // per staged row
    int32_t jj[KMAX];
    float w[KMAX], dd[KMAX], sj[KMAX];
    int32_t cnt, rt, pad[2];
};
template <int CPR, int KMAX, int LEAD>  // LEAD: chunks staged before the members (fwd 1 own row, bwd 2 grad halves)
struct PoolRing {
    static constexpr int SROW = (LEAD + KMAX) * CPR;  // uint4 chunks per staged row
    static constexpr size_t kRowBytes = size_t(SROW) * 16 + sizeof(PoolMeta<KMAX>);
    static constexpr size_t kWarpBytes = 2 * PoolGeo<CPR>::RPW * kRowBytes;
    static constexpr size_t kBytes = PoolGeo<CPR>::WARPS * kWarpBytes;
};

// Pool indices of one row spread over its LPR lanes: lane sl holds members
// sl, sl + LPR, ... (MPL per lane); loaded one round ahead of their gathers.
template <int CPR, int KMAX>
struct PoolLaneIdx {
    static constexpr int LPR = PoolGeo<CPR>::LPR, MPL = (KMAX + LPR - 1) / LPR;
    int j[MPL];
    double d[MPL];
    int cnt, rt;
    __device__ __forceinline__ void load(const int32_t* pool_idx, const double* pool_dist, const int32_t* pool_cnt,
                                         const int32_t* retained, int64_t row, int k_m, bool ok, int sl) {
#pragma unroll
        for (int i = 0; i < MPL; ++i) {
            const int t = sl + i * LPR;
            const bool v = ok && t < k_m;
            j[i] = v ? __ldg(pool_idx + row * k_m + t) : 0;
            d[i] = v ? __ldg(pool_dist + row * k_m + t) : 0.0;
        }
        cnt = ok ? __ldg(pool_cnt + row) : 0;
        rt = ok ? __ldg(retained + row) : 0;
    }
};

// Issue the gathers of one row into a stage slot: LEAD chunks from `lead_src`
// (16-byte chunk pointer of the row's own data), member chunks (zero-filled
// past the row's count, up to the warp's largest count `tmax`), metadata.
// softmax(-p * dist) weights as merging.cpp:121-149: max, exp, sum in member
// order, normalise (the same operation order as the per-thread form).
template <int CPR, int KMAX, int LEAD>
__device__ __forceinline__ void pool_issue_row(uint8_t* slot, const PoolLaneIdx<CPR, KMAX>& ix, float p, bool ok,
                                               int tmax, const uint4* lead_src, const uint4* fb, const float* sb,
                                               int lane) {
    using G = PoolGeo<CPR>;
    using Rg = PoolRing<CPR, KMAX, LEAD>;
    constexpr int MPL = PoolLaneIdx<CPR, KMAX>::MPL;
    const int sl = lane % G::LPR, base = lane - sl;
    uint4* ch16 = reinterpret_cast<uint4*>(slot);
    PoolMeta<KMAX>* m = reinterpret_cast<PoolMeta<KMAX>*>(slot + size_t(Rg::SROW) * 16);
    const int cnt = ok ? ix.cnt : 0;
    float e[MPL], dd[MPL];
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
        const int t = sl + i * G::LPR;
        dd[i] = t < cnt ? float(ix.d[i]) : 0.f;
        if (t < cnt) mx = fmaxf(mx, -p * dd[i]);
    }
#pragma unroll
    for (int o = G::LPR / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
    for (int i = 0; i < MPL; ++i) e[i] = (sl + i * G::LPR) < cnt ? __expf(-p * dd[i] - mx) : 0.f;
    float l = 0.f;  // sum in member order (every lane of the row gets the same value)
#pragma unroll
    for (int t = 0; t < KMAX; ++t) l += __shfl_sync(0xffffffffu, e[t / G::LPR], base + t % G::LPR);
    const float il = cnt > 0 ? 1.f / l : 0.f;
#pragma unroll
    for (int i = 0; i < MPL; ++i) {
        const int t = sl + i * G::LPR;
        if (t < KMAX) {
            m->jj[t] = t < cnt ? ix.j[i] : 0;
            m->w[t] = e[i] * il;
            m->dd[t] = dd[i];
            if (t < cnt) cp_async4(&m->sj[t], sb + ix.j[i]);
            else m->sj[t] = 0.f;
        }
    }
    if (sl == 0) {
        m->cnt = ok ? cnt : -1;
        m->rt = ix.rt;
    }
    if (ok) {
#pragma unroll
        for (int cc = 0; cc < G::CPL; ++cc) {
            const int ch = sl + cc * G::LPR;
#pragma unroll
            for (int l2 = 0; l2 < LEAD; ++l2) cp_async16(ch16 + l2 * CPR + ch, lead_src + l2 * CPR + ch);
        }
    }
#pragma unroll
    for (int t = 0; t < KMAX; ++t) {
        if (t >= tmax) break;  // warp-uniform
        const int jt = __shfl_sync(0xffffffffu, ix.j[t / G::LPR], base + t % G::LPR);
        const uint32_t nb = t < cnt ? 16u : 0u;
#pragma unroll
        for (int cc = 0; cc < G::CPL; ++cc) {
            const int ch = sl + cc * G::LPR;
            cp_async16_zfill(ch16 + (LEAD + t) * CPR + ch, fb + int64_t(nb ? jt : 0) * CPR + ch, nb);
        }
    }
}

template <int CPR, int KMAX>
__global__ void __launch_bounds__(PoolGeo<CPR>::WARPS * 32) pool_fwd_v3_kernel(
    const __nv_bfloat16* __restrict__ feats, const float* __restrict__ scores, const float* __restrict__ p_merge,
    const int32_t* __restrict__ retained, const int32_t* __restrict__ pool_idx,
    const double* __restrict__ pool_dist, const int32_t* __restrict__ pool_cnt, int64_t batch, int64_t n,
    int64_t r, int k_m, __nv_bfloat16* __restrict__ out) {
    using G = PoolGeo<CPR>;
    using Rg = PoolRing<CPR, KMAX, 1>;
    extern __shared__ __align__(16) uint8_t pool_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / G::LPR, sl = lane % G::LPR;
    uint8_t* ring = pool_smem + size_t(warp) * Rg::kWarpBytes;
    const int64_t total = batch * r;
    const int64_t GW = int64_t(gridDim.x) * G::WARPS;
    const float p = *p_merge;
    auto slot_of = [&](int stage) { return ring + size_t(stage * G::RPW + sub) * Rg::kRowBytes; };
    auto issue = [&](int64_t rd, int stage, const PoolLaneIdx<CPR, KMAX>& ix) {
        const int64_t row = rd * G::RPW + sub;
        const bool ok = row < total;
        const int64_t b = ok ? row / r : 0;
        const uint4* fb = reinterpret_cast<const uint4*>(feats + b * n * CPR * 8);
        const int tmax = __reduce_max_sync(0xffffffffu, ok ? ix.cnt : 0);
        pool_issue_row<CPR, KMAX, 1>(slot_of(stage), ix, p, ok, tmax, fb + int64_t(ix.rt) * CPR, fb,
                                     scores + b * n, lane);
    };
    int64_t rd = int64_t(blockIdx.x) * G::WARPS + warp;
    const int64_t nrounds = (total + G::RPW - 1) / G::RPW;
    PoolLaneIdx<CPR, KMAX> ix;
    {
        const int64_t row = rd * G::RPW + sub;
        ix.load(pool_idx, pool_dist, pool_cnt, retained, row, k_m, rd < nrounds && row < total, sl);
    }
    if (rd < nrounds) issue(rd, 0, ix);
    cp_async_commit();
    {
        const int64_t row = (rd + GW) * G::RPW + sub;
        ix.load(pool_idx, pool_dist, pool_cnt, retained, row, k_m, rd + GW < nrounds && row < total, sl);
    }
    for (int k = 0; rd < nrounds; ++k, rd += GW) {
        const int cur = k & 1;
        if (rd + GW < nrounds) issue(rd + GW, cur ^ 1, ix);
        cp_async_commit();
        {
            const int64_t row = (rd + 2 * GW) * G::RPW + sub;
            ix.load(pool_idx, pool_dist, pool_cnt, retained, row, k_m, rd + 2 * GW < nrounds && row < total, sl);
        }
        cp_async_wait<1>();
        __syncwarp();
        const uint8_t* slot = slot_of(cur);
        const uint4* src = reinterpret_cast<const uint4*>(slot);
        const PoolMeta<KMAX>* m = reinterpret_cast<const PoolMeta<KMAX>*>(slot + size_t(Rg::SROW) * 16);
        const int cnt = m->cnt;
        const int tmax = __reduce_max_sync(0xffffffffu, cnt);
        {
            const int64_t row = rd * G::RPW + sub;
            uint4* o = reinterpret_cast<uint4*>(out + (cnt >= 0 ? row : 0) * 2 * CPR * 8);
#pragma unroll
            for (int cc = 0; cc < G::CPL; ++cc) {
                const int ch = sl + cc * G::LPR;
                float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int t = 0; t < KMAX; ++t) {
                    if (t >= tmax) break;  // warp-uniform; members past the row's count are zero-filled
                    const float g = t < cnt ? m->w[t] * m->sj[t] : 0.f;
                    float f[8];
                    bf16x8_to_f32(src[(1 + t) * CPR + ch], f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = fmaf(g, f[i], acc[i]);
                }
                if (cnt >= 0) {
                    o[ch] = src[ch];
                    o[CPR + ch] = f32_to_bf16x8(acc);
                }
            }
        }
        __syncwarp();  // slot `cur` is reissued next round
    }
    cp_async_wait<0>();
}

template <int CPR, int KMAX>
__global__ void __launch_bounds__(PoolGeo<CPR>::WARPS * 32) pool_bwd_v3_kernel(
    const __nv_bfloat16* __restrict__ feats, const float* __restrict__ scores, const float* __restrict__ p_merge,
    const int32_t* __restrict__ retained, const int32_t* __restrict__ pool_idx,
    const double* __restrict__ pool_dist, const int32_t* __restrict__ pool_cnt, int64_t batch, int64_t n,
    int64_t r, int k_m, const __nv_bfloat16* __restrict__ dout, __nv_bfloat16* __restrict__ dfeats,
    float* __restrict__ dscores, float* __restrict__ dp_part) {
    using G = PoolGeo<CPR>;
    using Rg = PoolRing<CPR, KMAX, 2>;
    extern __shared__ __align__(16) uint8_t pool_smem[];
    __shared__ float red[G::WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / G::LPR, sl = lane % G::LPR;
    uint8_t* ring = pool_smem + size_t(warp) * Rg::kWarpBytes;
    const int64_t total = batch * r;
    const int64_t GW = int64_t(gridDim.x) * G::WARPS;
    const float p = *p_merge;
    auto slot_of = [&](int stage) { return ring + size_t(stage * G::RPW + sub) * Rg::kRowBytes; };
    auto issue = [&](int64_t rd, int stage, const PoolLaneIdx<CPR, KMAX>& ix) {
        const int64_t row = rd * G::RPW + sub;
        const bool ok = row < total;
        const int64_t b = ok ? row / r : 0;
        const uint4* fb = reinterpret_cast<const uint4*>(feats + b * n * CPR * 8);
        const uint4* gr = reinterpret_cast<const uint4*>(dout + (ok ? row : 0) * 2 * CPR * 8);
        const int tmax = __reduce_max_sync(0xffffffffu, ok ? ix.cnt : 0);
        pool_issue_row<CPR, KMAX, 2>(slot_of(stage), ix, p, ok, tmax, gr, fb, scores + b * n, lane);
    };
    float dp = 0.f;
    int64_t rd = int64_t(blockIdx.x) * G::WARPS + warp;
    const int64_t nrounds = (total + G::RPW - 1) / G::RPW;
    PoolLaneIdx<CPR, KMAX> ix;
    {
        const int64_t row = rd * G::RPW + sub;
        ix.load(pool_idx, pool_dist, pool_cnt, retained, row, k_m, rd < nrounds && row < total, sl);
    }
    if (rd < nrounds) issue(rd, 0, ix);
    cp_async_commit();
    {
        const int64_t row = (rd + GW) * G::RPW + sub;
        ix.load(pool_idx, pool_dist, pool_cnt, retained, row, k_m, rd + GW < nrounds && row < total, sl);
    }
    for (int k = 0; rd < nrounds; ++k, rd += GW) {
        const int cur = k & 1;
        if (rd + GW < nrounds) issue(rd + GW, cur ^ 1, ix);
        cp_async_commit();
        {
            const int64_t row = (rd + 2 * GW) * G::RPW + sub;
            ix.load(pool_idx, pool_dist, pool_cnt, retained, row, k_m, rd + 2 * GW < nrounds && row < total, sl);
        }
        cp_async_wait<1>();
        __syncwarp();
        const uint8_t* slot = slot_of(cur);
        const uint4* src = reinterpret_cast<const uint4*>(slot);
        const PoolMeta<KMAX>* m = reinterpret_cast<const PoolMeta<KMAX>*>(slot + size_t(Rg::SROW) * 16);
        const int cnt = m->cnt;
        const bool valid = cnt >= 0;
        const int64_t row = rd * G::RPW + sub;
        const int64_t b = valid ? row / r : 0;
        uint4* dfb = reinterpret_cast<uint4*>(dfeats + b * n * CPR * 8);
        float dot[KMAX];
#pragma unroll
        for (int t = 0; t < KMAX; ++t) dot[t] = 0.f;
        const int tmax = __reduce_max_sync(0xffffffffu, cnt);
        {
            const int64_t rt = valid ? m->rt : 0;
#pragma unroll
            for (int cc = 0; cc < G::CPL; ++cc) {
                const int ch = sl + cc * G::LPR;
                if (valid) dfb[rt * CPR + ch] = src[ch];
                float go[8];
                bf16x8_to_f32(src[CPR + ch], go);
#pragma unroll
                for (int t = 0; t < KMAX; ++t) {
                    if (t >= tmax) break;  // warp-uniform; members past the row's count are zero-filled
                    const float kt = t < cnt ? m->w[t] * m->sj[t] : 0.f;
                    float f[8], df[8];
                    bf16x8_to_f32(src[(2 + t) * CPR + ch], f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        dot[t] = fmaf(go[i], f[i], dot[t]);
                        df[i] = go[i] * kt;
                    }
                    if (t < cnt) dfb[int64_t(m->jj[t]) * CPR + ch] = f32_to_bf16x8(df);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < KMAX; ++t)
#pragma unroll
            for (int o = G::LPR / 2; o > 0; o >>= 1) dot[t] += __shfl_xor_sync(0xffffffffu, dot[t], o);
        if (valid && sl == 0) {
            float* dsb = dscores + b * n;
            dsb[m->rt] = 0.f;
            float wdot = 0.f;
#pragma unroll
            for (int t = 0; t < KMAX; ++t)
                if (t < cnt) {
                    dsb[m->jj[t]] = m->w[t] * dot[t];
                    wdot = fmaf(m->w[t], m->sj[t] * dot[t], wdot);
                }
#pragma unroll
            for (int t = 0; t < KMAX; ++t)
                if (t < cnt) dp = fmaf(m->w[t] * (m->sj[t] * dot[t] - wdot), -m->dd[t], dp);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    dp = warp_sum(dp);
    if (lane == 0) red[warp] = dp;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int i = 0; i < G::WARPS; ++i) s += red[i];
        dp_part[blockIdx.x] = s;
    }
}

// persistent grid: resident blocks per SM x SMs (never more blocks than rounds)
template <typename K>
static int pool_v3_grid(K kern, size_t smem, int warps, int64_t rounds, unsigned& nb) {
    static_assert(sizeof(K) > 0, "");
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return fail(AFFMAE_ECUDA, std::string("pool: ") + cudaGetErrorString(e));
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
    if (occ < 1) return fail(AFFMAE_EUNSUPPORTED, "pool: kernel does not fit on an SM");
    const int64_t want = (rounds + warps - 1) / warps;
    nb = unsigned(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(occ) * kNumSMs)));
    return AFFMAE_OK;
}

template <int CPR, int KMAX>
static int launch_pool_fwd_v3(const __nv_bfloat16* feats, const float* scores, const float* p_merge,
                              const int32_t* retained, const affmae_merge_plan* plan, int64_t batch, int64_t n,
                              int64_t r, int k_m, __nv_bfloat16* out, cudaStream_t st) {
    using G = PoolGeo<CPR>;
    auto kern = pool_fwd_v3_kernel<CPR, KMAX>;
    const size_t smem = PoolRing<CPR, KMAX, 1>::kBytes;
    unsigned nb = 0;
    int rc = pool_v3_grid(kern, smem, G::WARPS, (batch * r + G::RPW - 1) / G::RPW, nb);
    if (rc) return rc;
    kern<<<nb, G::WARPS * 32, smem, st>>>(feats, scores, p_merge, retained, plan->pool_idx, plan->pool_dist,
                                          plan->pool_cnt, batch, n, r, k_m, out);
    AFFMAE_LAUNCH_CHECK("pool_fwd_v3_kernel");
    return AFFMAE_OK;
}
template <int CPR>
static int launch_pool_fwd_v2(const __nv_bfloat16* feats, const float* scores, const float* p_merge,
                              const int32_t* retained, const affmae_merge_plan* plan, int64_t batch, int64_t n,
                              int64_t r, int k_m, __nv_bfloat16* out, cudaStream_t st) {
    return k_m <= 8 ? launch_pool_fwd_v3<CPR, 8>(feats, scores, p_merge, retained, plan, batch, n, r, k_m, out, st)
                    : launch_pool_fwd_v3<CPR, 16>(feats, scores, p_merge, retained, plan, batch, n, r, k_m, out, st);
}
template <int CPR, int KMAX>
static int launch_pool_bwd_v3(const __nv_bfloat16* feats, const float* scores, const float* p_merge,
                              const int32_t* retained, const affmae_merge_plan* plan, int64_t batch, int64_t n,
                              int64_t r, int k_m, const __nv_bfloat16* dout, __nv_bfloat16* dfeats,
                              float* dscores, float* part, cudaStream_t st, unsigned& nb) {
    using G = PoolGeo<CPR>;
    auto kern = pool_bwd_v3_kernel<CPR, KMAX>;
    const size_t smem = PoolRing<CPR, KMAX, 2>::kBytes;
    int rc = pool_v3_grid(kern, smem, G::WARPS, (batch * r + G::RPW - 1) / G::RPW, nb);
    if (rc) return rc;
    kern<<<nb, G::WARPS * 32, smem, st>>>(feats, scores, p_merge, retained, plan->pool_idx, plan->pool_dist,
                                          plan->pool_cnt, batch, n, r, k_m, dout, dfeats, dscores, part);
    AFFMAE_LAUNCH_CHECK("pool_bwd_v3_kernel");
    return AFFMAE_OK;
}
template <int CPR>
static int launch_pool_bwd_v2(const __nv_bfloat16* feats, const float* scores, const float* p_merge,
                              const int32_t* retained, const affmae_merge_plan* plan, int64_t batch, int64_t n,
                              int64_t r, int k_m, const __nv_bfloat16* dout, __nv_bfloat16* dfeats,
                              float* dscores, float* part, cudaStream_t st, unsigned& nb) {
    pool_bwd_zero_vec_kernel<CPR><<<unsigned((batch * n + 255) / 256), 256, 0, st>>>(plan->row_of, batch * n,
                                                                                    dfeats, dscores);
    AFFMAE_LAUNCH_CHECK("pool_bwd_zero_vec_kernel");
    return k_m <= 8 ? launch_pool_bwd_v3<CPR, 8>(feats, scores, p_merge, retained, plan, batch, n, r, k_m, dout,
                                                 dfeats, dscores, part, st, nb)
                    : launch_pool_bwd_v3<CPR, 16>(feats, scores, p_merge, retained, plan, batch, n, r, k_m, dout,
                                                  dfeats, dscores, part, st, nb);
}

// ===================================================================== host
struct SelWs {
    uint64_t* keys[2];
    uint32_t* vals[2];
    uint32_t* hist;
    uint8_t* keep;
    size_t bytes;
};
static SelWs carve_sel(int64_t batch, int64_t n, void* base) {
    SelWs w{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* q = p ? p + off : nullptr;
        off += al256(bytes);
        return q;
    };
    const size_t e = size_t(batch) * n;
    w.keys[0] = reinterpret_cast<uint64_t*>(take(e * 8));
    w.keys[1] = reinterpret_cast<uint64_t*>(take(e * 8));
    w.vals[0] = reinterpret_cast<uint32_t*>(take(e * 4));
    w.vals[1] = reinterpret_cast<uint32_t*>(take(e * 4));
    w.hist = reinterpret_cast<uint32_t*>(take(radix_hist_elems(int64_t(e)) * 4));
    w.keep = reinterpret_cast<uint8_t*>(take(e));
    w.bytes = off;
    return w;
}

int64_t retained_count_impl(int64_t n, double d_s) {
    if (!(d_s > 0.0 && d_s <= 1.0)) return -2;
    int64_t k = int64_t(std::floor(d_s * double(n) + 0.5));
    if (k > n) k = n;
    return k < 1 ? 1 : k;
}

size_t select_retained_workspace(int64_t batch, int64_t n) {
    if (batch < 0 || n < 1) return 0;
    return carve_sel(batch, n, nullptr).bytes;
}

int select_retained(const float* scores, int64_t batch, int64_t n, double d_s, int32_t* retained,
                    void* workspace, size_t ws_bytes, void* stream) {
    const int64_t r = retained_count_impl(n, d_s);
    if (r < 0) return fail(AFFMAE_ECONFIG, "retained_count: d_s must be in (0, 1]");
    if (n < 1) return fail(AFFMAE_ECONFIG, "select_retained: empty score set");
    if (!scores || !retained) return fail(AFFMAE_ECONFIG, "select_retained: null pointer");
    SelWs w = carve_sel(batch, n, workspace);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "select_retained: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    if (n <= kSegSortMax) {
        const size_t smem = size_t(n) * 4;
        // per-call (the attribute is per device and the call is a cheap host-side set)
        AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(select_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               int(kSegSortMax * 4)));
        select_topk_kernel<<<unsigned(batch), kSelWarps * 32, smem, st>>>(scores, n, r, retained);
        AFFMAE_LAUNCH_CHECK("select_topk_kernel");
        return AFFMAE_OK;
    }
    score_keys_kernel<<<blocks_of(batch * n), 256, 0, st>>>(scores, batch, n, w.keys[0], w.vals[0]);
    uint64_t* k = w.keys[0];
    uint32_t* v = w.vals[0];
    int rc = segmented_sort(k, v, w.keys[1], w.vals[1], batch, n, 32 + bits_for(batch), w.hist, st);
    if (rc) return rc;
    keep_flags_kernel<<<blocks_of(batch * n), 256, 0, st>>>(v, batch, n, r, w.keep);
    compact_kernel<<<unsigned(batch), 1024, 0, st>>>(w.keep, n, r, retained);
    AFFMAE_LAUNCH_CHECK("select_retained");
    return AFFMAE_OK;
}

struct PlanWs {
    GridPrm* prm;
    int32_t* ret_pos;
    int32_t* cell_off;
    int32_t* cell_cur;
    int32_t* items;
    float2* item_xy;
    int32_t* best_of;
    double* d2_of;
    int32_t* pool_off;
    int32_t* pool_cur;
    double* ldist;
    int32_t* lidx;
    size_t bytes;
};

static int grid_side(int64_t r) {
    int g = int(std::ceil(std::sqrt(double(r))));
    return g < 1 ? 1 : g;
}

static PlanWs carve_plan(int64_t batch, int64_t n, int64_t r, void* base) {
    PlanWs w{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* q = p ? p + off : nullptr;
        off += al256(bytes);
        return q;
    };
    const int64_t g = grid_side(r);
    const size_t cells = size_t(batch) * (g * g + 1);
    w.prm = reinterpret_cast<GridPrm*>(take(size_t(batch) * sizeof(GridPrm)));
    w.ret_pos = reinterpret_cast<int32_t*>(take(size_t(batch) * n * 4));
    w.cell_off = reinterpret_cast<int32_t*>(take(cells * 4));
    w.cell_cur = reinterpret_cast<int32_t*>(take(cells * 4));
    w.items = reinterpret_cast<int32_t*>(take(size_t(batch) * r * 4));
    w.item_xy = reinterpret_cast<float2*>(take(size_t(batch) * r * 8));
    w.best_of = reinterpret_cast<int32_t*>(take(size_t(batch) * n * 4));
    w.d2_of = reinterpret_cast<double*>(take(size_t(batch) * n * 8));
    w.pool_off = reinterpret_cast<int32_t*>(take(size_t(batch) * (r + 1) * 4));
    w.pool_cur = reinterpret_cast<int32_t*>(take(size_t(batch) * (r + 1) * 4));
    w.ldist = reinterpret_cast<double*>(take(size_t(batch) * n * 8));
    w.lidx = reinterpret_cast<int32_t*>(take(size_t(batch) * n * 4));
    w.bytes = off;
    return w;
}

size_t merge_plan_workspace(int64_t batch, int64_t n, int64_t r) {
    if (batch < 0 || n < 1 || r < 1) return 0;
    return carve_plan(batch, n, r, nullptr).bytes;
}

int merge_plan_build(const float* coords, const int32_t* retained, int64_t batch, int64_t n, int64_t r,
                     int k_m, affmae_merge_plan* plan, void* workspace, size_t ws_bytes, void* stream) {
    if (r < 1) return fail(AFFMAE_ECONFIG, "merge_plan: retained set empty");
    if (k_m < 1) return fail(AFFMAE_ECONFIG, "merge_plan: k_m must be >= 1");
    if (k_m > kMaxKm) return fail(AFFMAE_EUNSUPPORTED, "merge_plan: k_m > 16 not compiled");
    if (r > n) return fail(AFFMAE_ECONFIG, "merge_plan: more retained than tokens");
    if (!coords || !retained || !plan || !plan->target || !plan->pool_idx || !plan->pool_dist ||
        !plan->pool_cnt || !plan->row_of)
        return fail(AFFMAE_ECONFIG, "merge_plan: null pointer");
    PlanWs w = carve_plan(batch, n, r, workspace);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "merge_plan: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const int g = grid_side(r);
    const int64_t cells = int64_t(g) * g + 1;
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.ret_pos, 0xFF, size_t(batch) * n * 4, st));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.cell_off, 0, size_t(batch) * cells * 4, st));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.cell_cur, 0, size_t(batch) * cells * 4, st));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.pool_off, 0, size_t(batch) * (r + 1) * 4, st));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.pool_cur, 0, size_t(batch) * (r + 1) * 4, st));
    grid_prm_kernel<<<unsigned(batch), 256, 0, st>>>(coords, n, g, w.prm);
    mark_retained_kernel<<<blocks_of(batch * r), 256, 0, st>>>(retained, batch, n, r, w.ret_pos);
    cell_count_kernel<<<blocks_of(batch * r), 256, 0, st>>>(coords, retained, batch, n, r, g, w.prm, w.cell_off);
    seg_scan_kernel<<<unsigned(batch), 1024, 0, st>>>(w.cell_off, cells);
    cell_fill_kernel<<<blocks_of(batch * r), 256, 0, st>>>(coords, retained, batch, n, r, g, w.prm,
                                                           w.cell_off, w.cell_cur, w.items, w.item_xy);
    assign_kernel<<<blocks_of(batch * n, 128), 128, 0, st>>>(coords, retained, w.ret_pos, batch, n, r, g, w.prm,
                                                        w.cell_off, w.items, w.item_xy, plan->target, w.best_of,
                                                        w.d2_of, w.pool_off);
    seg_scan_kernel<<<unsigned(batch), 1024, 0, st>>>(w.pool_off, r + 1);
    pool_fill_kernel<<<blocks_of(batch * n), 256, 0, st>>>(w.best_of, w.d2_of, batch, n, r, w.pool_off,
                                                           w.pool_cur, w.ldist, w.lidx);
    pool_topk_kernel<<<blocks_of(batch * r, 256), 256, 0, st>>>(w.pool_off, batch, n, r, k_m, w.ldist, w.lidx,
                                                                     plan->pool_idx, plan->pool_dist,
                                                                     plan->pool_cnt, plan->row_of, retained);
    AFFMAE_LAUNCH_CHECK("merge_plan");
    return AFFMAE_OK;
}

int merge_pool_fwd(const affmae_bf16* feats, const float* scores, const float* p_merge,
                   const int32_t* retained, const affmae_merge_plan* plan, int64_t batch, int64_t n,
                   int64_t r, int64_t dim, int k_m, affmae_bf16* out, void* stream) {
    if (!feats || !scores || !p_merge || !retained || !plan || !out)
        return fail(AFFMAE_ECONFIG, "merge_pool: null pointer");
    if (dim < 2 || dim % 2) return fail(AFFMAE_EUNSUPPORTED, "merge_pool: dim must be even");
    if (k_m < 1 || k_m > kMaxKm) return fail(AFFMAE_EUNSUPPORTED, "merge_pool: k_m must be in [1, 16]");
    if (batch * r == 0) return AFFMAE_OK;
    {
        const auto* f = reinterpret_cast<const __nv_bfloat16*>(feats);
        auto* o = reinterpret_cast<__nv_bfloat16*>(out);
        cudaStream_t st = as_stream(stream);
        switch (dim) {
            case 64: return launch_pool_fwd_v2<8>(f, scores, p_merge, retained, plan, batch, n, r, k_m, o, st);
            case 128: return launch_pool_fwd_v2<16>(f, scores, p_merge, retained, plan, batch, n, r, k_m, o, st);
            case 256: return launch_pool_fwd_v2<32>(f, scores, p_merge, retained, plan, batch, n, r, k_m, o, st);
            case 512: return launch_pool_fwd_v2<64>(f, scores, p_merge, retained, plan, batch, n, r, k_m, o, st);
            default: break;
        }
    }
    pool_fwd_kernel<<<blocks_of(batch * r * 32), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(feats), scores, p_merge, retained, plan->pool_idx,
        plan->pool_dist, plan->pool_cnt, batch, n, r, int(dim), k_m, reinterpret_cast<__nv_bfloat16*>(out));
    AFFMAE_LAUNCH_CHECK("pool_fwd_kernel");
    return AFFMAE_OK;
}

size_t merge_pool_bwd_workspace(int64_t batch, int64_t r) {
    return al256(size_t(blocks_of(batch * r * 32)) * 4 + 4);  // >= every variant's block count
}

int merge_pool_bwd(const affmae_bf16* feats, const float* scores, const float* p_merge,
                   const int32_t* retained, const affmae_merge_plan* plan, int64_t batch, int64_t n,
                   int64_t r, int64_t dim, int k_m, const affmae_bf16* dout, affmae_bf16* dfeats,
                   float* dscores, float* dp, void* workspace, size_t ws_bytes, void* stream) {
    if (!feats || !scores || !p_merge || !retained || !plan || !dout || !dfeats || !dscores || !dp)
        return fail(AFFMAE_ECONFIG, "merge_pool bwd: null pointer");
    if (dim < 2 || dim % 2) return fail(AFFMAE_EUNSUPPORTED, "merge_pool: dim must be even");
    if (k_m < 1 || k_m > kMaxKm) return fail(AFFMAE_EUNSUPPORTED, "merge_pool: k_m must be in [1, 16]");
    if (!workspace || ws_bytes < merge_pool_bwd_workspace(batch, r))
        return fail(AFFMAE_ECONFIG, "merge_pool bwd: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    float* part = static_cast<float*>(workspace);
    {
        const auto* f = reinterpret_cast<const __nv_bfloat16*>(feats);
        const auto* g = reinterpret_cast<const __nv_bfloat16*>(dout);
        auto* df = reinterpret_cast<__nv_bfloat16*>(dfeats);
        unsigned nb2 = 0;
        int rc = -1;
        switch (dim) {
            case 64: rc = launch_pool_bwd_v2<8>(f, scores, p_merge, retained, plan, batch, n, r, k_m, g, df, dscores, part, st, nb2); break;
            case 128: rc = launch_pool_bwd_v2<16>(f, scores, p_merge, retained, plan, batch, n, r, k_m, g, df, dscores, part, st, nb2); break;
            case 256: rc = launch_pool_bwd_v2<32>(f, scores, p_merge, retained, plan, batch, n, r, k_m, g, df, dscores, part, st, nb2); break;
            case 512: rc = launch_pool_bwd_v2<64>(f, scores, p_merge, retained, plan, batch, n, r, k_m, g, df, dscores, part, st, nb2); break;
            default: break;
        }
        if (rc > 0) return rc;
        if (rc == 0) {
            dp_reduce_kernel<<<1, 1024, 0, st>>>(part, int(nb2), dp);
            AFFMAE_LAUNCH_CHECK("dp_reduce_kernel");
            return AFFMAE_OK;
        }
    }
    const unsigned nb = blocks_of(batch * r * 32);
    pool_bwd_zero_kernel<<<blocks_of(batch * n * 32), 256, 0, st>>>(
        plan->row_of, batch * n, int(dim), reinterpret_cast<__nv_bfloat16*>(dfeats), dscores);
    pool_bwd_kernel<<<nb, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(feats), scores, p_merge,
                                        retained, plan->pool_idx, plan->pool_dist, plan->pool_cnt, batch,
                                        n, r, int(dim), k_m, reinterpret_cast<const __nv_bfloat16*>(dout),
                                        reinterpret_cast<__nv_bfloat16*>(dfeats), dscores, part);
    dp_reduce_kernel<<<1, 1024, 0, st>>>(part, int(nb), dp);
    AFFMAE_LAUNCH_CHECK("pool_bwd_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
