// Cluster / neighbour index builder, batched and bit-exact with the reference:
//   sfc_order            proj/src/geometry.cpp:57-106
//   balanced_clusters    proj/src/geometry.cpp:108-131
//   cluster_neighborhood proj/src/geometry.cpp:133-186
//   knn                  proj/src/geometry.cpp:188-216
//
// Bit-exactness.  Every floating-point step the reference takes in binary64 is
// repeated in binary64 with explicit round-to-nearest intrinsics (no FMA
// contraction): coordinate extents and gaps (differences of binary32 values,
// exact), the quantisation (x - xmin) * scale with llround (half away from
// zero), centroids as sequential member-order sums times 1.0/|c|, and
// d^2 = dx*dx + dy*dy.  ceil(log2(.)) emulates a correctly rounded log2 (the
// glibc behaviour) exactly except within half an ulp of the rounding boundary.
// Ordering: a stable LSD radix sort (sort.cuh) on (image, key) reproduces
// std::stable_sort; the neighbour selection keeps the (d^2, j) order of
// std::partial_sort and puts the own cluster first (geometry.cpp:166-172).
#include <cmath>

#include "sort.cuh"

namespace affmae_b200 {

// hilbert_index, proj/src/geometry.cpp:15-30
__host__ __device__ __forceinline__ uint64_t hilbert(uint32_t n, uint32_t x, uint32_t y) {
    uint64_t d = 0;
    for (uint32_t s = n / 2; s > 0; s /= 2) {
        uint32_t rx = (x & s) ? 1u : 0u;
        uint32_t ry = (y & s) ? 1u : 0u;
        d += uint64_t(s) * uint64_t(s) * ((3u * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            uint32_t t = x;
            x = y;
            y = t;
        }
    }
    return d;
}

uint64_t hilbert_index_host(uint32_t n, uint32_t x, uint32_t y) { return hilbert(n, x, y); }

// ---------------------------------------------------------- sfc_order
__global__ void axis_keys_kernel(const float* __restrict__ coords, int64_t batch, int64_t n,
                                 uint64_t* __restrict__ keys, const int* __restrict__ run_flag) {
    if (run_flag && *run_flag == 0) return;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * n * 2) return;
    int64_t tok = i >> 1;
    int axis = int(i & 1);
    int64_t img = tok / n, j = tok - img * n;
    uint64_t seg = uint64_t(img) * 2 + axis;
    // segment-major layout: [img][axis][j]
    keys[(img * 2 + axis) * n + j] = (seg << 32) | float_order(coords[i]);
}

// min_gap: smallest positive gap between consecutive sorted values (0 if none)
__global__ void gap_kernel(const uint64_t* __restrict__ sorted, int64_t segs, int64_t n,
                           unsigned long long* __restrict__ gap_bits) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= segs * n) return;
    int64_t j = i % n;
    if (j == 0) return;
    double a = double(float_unorder(uint32_t(sorted[i - 1]))), b = double(float_unorder(uint32_t(sorted[i])));
    double d = __dsub_rn(b, a);
    if (d > 0.0) atomicMin(gap_bits + i / n, (unsigned long long)__double_as_longlong(d));
}

// min_gap without the axis sort (images of <= 16384 tokens): per (image, axis), one block
// takes min / max, drops every value into one of 4096 equal-width buckets (ordered-bit atomic
// min / max in shared memory; the bucket map is monotone), and reads the gaps between
// consecutive non-empty buckets -- each such pair of bucket max / next bucket min IS a pair
// of consecutive distinct sorted values, so every candidate is an exact min_gap candidate.
// Gaps between distinct values inside one bucket are invisible to it: such a bucket raises
// `hard`, and the (gated) segmented sort then runs and min-merges the exact gaps.  Lattice
// coordinates (patch centres) never share a bucket, so the sort is skipped.
constexpr int kAxisBuckets = 4096;
__global__ void __launch_bounds__(1024) axis_stats_kernel(const float* __restrict__ coords, int64_t n,
                                                          float2* __restrict__ minmax,
                                                          unsigned long long* __restrict__ gap_bits,
                                                          int* __restrict__ hard) {
    __shared__ uint32_t bmin[kAxisBuckets], bmax[kAxisBuckets];
    __shared__ float rlo[32], rhi[32];
    __shared__ uint32_t rlast[32];
    __shared__ double rgap[32];
    __shared__ int rhard;
    const int seg = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const float* c = coords + int64_t(seg >> 1) * n * 2 + (seg & 1);
    // each thread holds a contiguous chunk of <= 16 tokens in registers (one global read;
    // contiguous chunks put the lanes of a warp in different raster rows, so the bucket atomics
    // below do not pile onto one address -- a raster row shares its y)
    constexpr int kChunk = kSegSortMax / 1024;
    const int chunk = int((n + blockDim.x - 1) / blockDim.x);
    const int64_t j0 = int64_t(t) * chunk;
    float vals[kChunk];
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
        vals[i] = 0.f;
        if (i < chunk && j0 + i < n) {
            vals[i] = c[2 * (j0 + i)];
            lo = fminf(lo, vals[i]);
            hi = fmaxf(hi, vals[i]);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
        rlo[warp] = lo;
        rhi[warp] = hi;
    }
    for (int b = t; b < kAxisBuckets; b += blockDim.x) {
        bmin[b] = 0xffffffffu;
        bmax[b] = 0u;
    }
    if (t == 0) rhard = 0;
    __syncthreads();
    lo = rlo[0];
    hi = rhi[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
        lo = fminf(lo, rlo[w]);
        hi = fmaxf(hi, rhi[w]);
    }
    const float span = hi - lo, inv = span > 0.f ? float(kAxisBuckets) / span : 0.f;
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
        if (i < chunk && j0 + i < n) {
            const int b = min(kAxisBuckets - 1, int((vals[i] - lo) * inv));
            const uint32_t u = float_order(vals[i]);
            atomicMin(&bmin[b], u);
            atomicMax(&bmax[b], u);
        }
    }
    __syncthreads();
    // thread t: buckets [t*per, (t+1)*per): first / last value, gaps between its non-empty ones
    const int per = kAxisBuckets / int(blockDim.x);
    uint32_t first = 0u, last = 0u;
    double g = INFINITY;
    bool h = false;
    for (int b = t * per; b < (t + 1) * per; ++b) {
        if (bmax[b] == 0u) continue;  // empty (float_order of a real value is never 0)
        h |= bmin[b] != bmax[b];
        if (last) g = fmin(g, __dsub_rn(double(float_unorder(bmin[b])), double(float_unorder(last))));
        if (!first) first = bmin[b];
        last = bmax[b];
    }
    // exclusive max-scan of `last` over the threads: the previous non-empty value
    uint32_t inc = last;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = max(inc, y);
    }
    if (lane == 31) rlast[warp] = inc;
    __syncthreads();
    uint32_t prev = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) prev = 0u;
    for (int w = 0; w < warp; ++w) prev = max(prev, rlast[w]);
    if (first && prev) g = fmin(g, __dsub_rn(double(float_unorder(first)), double(float_unorder(prev))));
    for (int o = 16; o > 0; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (__any_sync(0xffffffffu, h) && lane == 0) rhard = 1;
    if (lane == 0) rgap[warp] = g;
    __syncthreads();
    if (t == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) g = fmin(g, rgap[w]);
        if (g > 0.0 && g < INFINITY) atomicMin(gap_bits + seg, (unsigned long long)__double_as_longlong(g));
        minmax[seg] = make_float2(lo, hi);
        if (rhard) atomicOr(hard, 1);
    }
}

struct SfcParams {
    double xmin, ymin, scale;
    uint32_t side;  // 0 -> identity order (n == 1 or all points coincide)
    uint32_t pad;
};

// ceil(log2(x)) for x >= 2 as a correctly rounded log2 followed by ceil
__device__ int ceil_log2_cr(double x) {
    int e = ilogb(x);
    double m = scalbn(x, -e);  // exact, in [1, 2)
    if (m == 1.0) return e;
    double u = scalbn(1.0, ilogb(double(e)) - 52);  // ulp of e
    return ((m - 1.0) * 1.4426950408889634 < 0.5 * u) ? e : e + 1;
}

// sfc_order quantisation parameters of image b (geometry.cpp:87-101) from its
// sorted axes and min gaps
__device__ SfcParams sfc_params(const uint64_t* __restrict__ sorted, const float2* __restrict__ minmax, int64_t b,
                                int64_t n, const unsigned long long* __restrict__ gap_bits) {
    SfcParams p{};
    double xmin, xmax, ymin, ymax;
    if (minmax) {  // axis statistics pass (axis_stats_kernel)
        const float2 mx = minmax[b * 2], my = minmax[b * 2 + 1];
        xmin = mx.x;
        xmax = mx.y;
        ymin = my.x;
        ymax = my.y;
    } else {  // ends of the sorted axes
        const uint64_t* xs = sorted + (b * 2) * n;
        const uint64_t* ys = sorted + (b * 2 + 1) * n;
        xmin = float_unorder(uint32_t(xs[0]));
        xmax = float_unorder(uint32_t(xs[n - 1]));
        ymin = float_unorder(uint32_t(ys[0]));
        ymax = float_unorder(uint32_t(ys[n - 1]));
    }
    double ex = __dsub_rn(xmax, xmin), ey = __dsub_rn(ymax, ymin);
    double extent = ex < ey ? ey : ex;
    p.xmin = xmin;
    p.ymin = ymin;
    if (n == 1 || extent <= 0.0) {
        p.side = 0;
    } else {
        unsigned long long gx = gap_bits[b * 2], gy = gap_bits[b * 2 + 1];
        double dgx = gx == ~0ull ? 0.0 : __longlong_as_double((long long)gx);
        double dgy = gy == ~0ull ? 0.0 : __longlong_as_double((long long)gy);
        double spacing = dgx < dgy ? dgy : dgx;
        if (spacing <= 0.0) spacing = extent;
        double arg = __dadd_rn(__ddiv_rn(extent, spacing), 1.0);
        if (2.0 > arg) arg = 2.0;
        int bb = ceil_log2_cr(arg);
        bb = bb < 1 ? 1 : (bb > 16 ? 16 : bb);
        p.side = 1u << bb;
        p.scale = __ddiv_rn(double(p.side - 1), extent);
    }
    return p;
}

// Hilbert keys; every thread derives its image's parameters (a few broadcast
// loads and binary64 ops) instead of a separate one-thread-per-image kernel.
__global__ void hilbert_keys_kernel(const float* __restrict__ coords, int64_t batch, int64_t n,
                                    const uint64_t* __restrict__ sorted_axes, const float2* __restrict__ minmax,
                                    const unsigned long long* __restrict__ gap_bits, uint64_t* __restrict__ keys,
                                    uint32_t* __restrict__ vals) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * n) return;
    int64_t b = i / n;
    const SfcParams p = sfc_params(sorted_axes, minmax, b, n, gap_bits);
    uint64_t key = 0;
    if (p.side) {
        double x = coords[2 * i], y = coords[2 * i + 1];
        uint32_t qx = uint32_t(llround(__dmul_rn(__dsub_rn(x, p.xmin), p.scale)));
        uint32_t qy = uint32_t(llround(__dmul_rn(__dsub_rn(y, p.ymin), p.scale)));
        key = hilbert(p.side, qx, qy);
    }
    keys[i] = (uint64_t(b) << 32) | key;
    vals[i] = uint32_t(i - b * n);
}

// ------------------------------------------------ clusters + neighbours
__global__ void perm_kernel(const uint32_t* __restrict__ sorted_vals, int64_t batch, ClusterShape cs,
                            int32_t* __restrict__ perm, int32_t* __restrict__ cluster_of) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * cs.n) return;
    int64_t b = i / cs.n;
    int pos = int(i - b * cs.n);
    int tok = int(sorted_vals[i]);
    perm[i] = tok;
    if (cluster_of) cluster_of[b * cs.n + tok] = cs.cluster_at(pos);
}

// perm + cluster_of + centroid in one pass, thread per cluster (the cluster's
// centroid = (sequential member-order sum) * (1.0 / |c|), geometry.cpp:140-150;
// curve positions are contiguous): the sorted token ids are read once.
__global__ void perm_centroid_kernel(const uint32_t* __restrict__ sorted_vals, const float* __restrict__ coords,
                                     int64_t batch, ClusterShape cs, int32_t* __restrict__ perm,
                                     int32_t* __restrict__ cluster_of, double2* __restrict__ cent) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * cs.c) return;
    const int64_t b = i / cs.c;
    const int k = int(i - b * cs.c);
    const int64_t base = b * cs.n + cs.off(k);
    const float2* xy = reinterpret_cast<const float2*>(coords) + b * cs.n;
    double sx = 0.0, sy = 0.0;
    const int len = cs.len(k);
    for (int j = 0; j < len; ++j) {
        const int tok = int(sorted_vals[base + j]);
        perm[base + j] = tok;
        cluster_of[b * cs.n + tok] = k;
        const float2 v = xy[tok];
        sx = __dadd_rn(sx, double(v.x));
        sy = __dadd_rn(sy, double(v.y));
    }
    const double inv = __ddiv_rn(1.0, double(len));
    cent[i] = make_double2(__dmul_rn(sx, inv), __dmul_rn(sy, inv));
}

constexpr int kMaxGroups = 8;

__device__ __forceinline__ bool pair_lt(double da, int ja, double db, int jb) {
    return da < db || (!(db < da) && ja < jb);
}

// Merges per-lane sorted top-G lists into the warp's top-G (ascending (d, j)).
// Register-only: the lane's list head is selected with unrolled compares.
template <int G>
__device__ __forceinline__ void warp_topk(double (&d)[G], int (&j)[G], int g, double* outd, int* outj) {
    int head = 0;
#pragma unroll
    for (int r = 0; r < G; ++r) {
        if (r >= g) break;
        double md = INFINITY;
        int mj = INT32_MAX;
#pragma unroll
        for (int q = 0; q < G; ++q)
            if (q == head && q < g) {
                md = d[q];
                mj = j[q];
            }
        double bd = md;
        int bj = mj;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double od = __shfl_xor_sync(0xffffffffu, bd, o);
            int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (pair_lt(od, oj, bd, bj)) {
                bd = od;
                bj = oj;
            }
        }
        if (head < g && md == bd && mj == bj) ++head;
        outd[r] = bd;
        outj[r] = bj;
    }
}

template <int G>
__device__ __forceinline__ void topk_insert(double (&d)[G], int (&j)[G], int g, double nd, int nj) {
    if (!pair_lt(nd, nj, d[g - 1], j[g - 1])) return;
    int p = g - 1;
    while (p > 0 && pair_lt(nd, nj, d[p - 1], j[p - 1])) {
        d[p] = d[p - 1];
        j[p] = j[p - 1];
        --p;
    }
    d[p] = nd;
    j[p] = nj;
}

// one warp per (image, cluster k): the G smallest (d^2, j) over all centroids,
// then own cluster first (proj/src/geometry.cpp:157-172)
__global__ void nbr_kernel(const double2* __restrict__ cent, int64_t batch, ClusterShape cs,
                           int32_t* __restrict__ nbr_cl) {
    const int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= batch * cs.c) return;
    int64_t b = w / cs.c;
    int k = int(w - b * cs.c);
    const double2* cb = cent + b * cs.c;
    const double2 ck = cb[k];
    const int g = cs.g;
    double d[kMaxGroups];
    int jj[kMaxGroups];
    for (int r = 0; r < kMaxGroups; ++r) {
        d[r] = INFINITY;
        jj[r] = INT32_MAX;
    }
    for (int j = lane; j < cs.c; j += 32) {
        double2 cj = cb[j];
        double dx = __dsub_rn(cj.x, ck.x), dy = __dsub_rn(cj.y, ck.y);
        double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        topk_insert<kMaxGroups>(d, jj, g, d2, j);
    }
    double od[kMaxGroups];
    int oj[kMaxGroups];
    warp_topk<kMaxGroups>(d, jj, g, od, oj);
    if (lane == 0) {
        int32_t* sel = nbr_cl + w * g;
        int ns = 0;
        sel[ns++] = k;
        for (int r = 0; r < g && ns < g; ++r)
            if (oj[r] != k) sel[ns++] = oj[r];
    }
}

// v2: one CTA per (image, block of clusters).  The image's centroids are
// staged in shared memory; each warp keeps a lane-local top-G in registers
// (branch-free insertion network, compile-time G) and merges with warp_topk.
// Same (d^2, j) order and own-first selection as nbr_kernel.
template <int G>
__device__ __forceinline__ void topk_push(double (&d)[G], int (&j)[G], double nd, int nj) {
#pragma unroll
    for (int p = 0; p < G; ++p) {
        if (pair_lt(nd, nj, d[p], j[p])) {
            const double td = d[p];
            const int tj = j[p];
            d[p] = nd;
            j[p] = nj;
            nd = td;
            nj = tj;
        }
    }
}
constexpr int kNbrWarps = 8, kNbrPerWarp = 4;
template <int G>
__global__ void __launch_bounds__(kNbrWarps * 32) nbr_v2_kernel(const double2* __restrict__ cent, ClusterShape cs,
                                                                 int32_t* __restrict__ nbr_cl) {
    // smem: binary64 centroids, their fp32 copies, the fp32 bounding box of every run of 32
    // clusters in curve order
    extern __shared__ double2 sc[];
    float2* sf = reinterpret_cast<float2*>(sc + cs.c);
    const int nchunk = (cs.c + 31) / 32;
    float4* sbox = reinterpret_cast<float4*>(sf + ((cs.c + 1) & ~1));
    __shared__ unsigned int smax;
    const int b = blockIdx.y;
    const double2* cb = cent + int64_t(b) * cs.c;
    if (threadIdx.x == 0) smax = 0u;
    __syncthreads();
    float lmax = 0.f;
    for (int i = threadIdx.x; i < cs.c; i += blockDim.x) {
        const double2 c = cb[i];
        sc[i] = c;
        sf[i] = make_float2(float(c.x), float(c.y));
        lmax = fmaxf(lmax, fmaxf(fabsf(float(c.x)), fabsf(float(c.y))));
    }
    atomicMax(&smax, __float_as_uint(lmax));  // non-negative floats order like their bits
    __syncthreads();
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int q = warp; q < nchunk; q += kNbrWarps) {
            const int j = q * 32 + lane;
            const float2 f = j < cs.c ? sf[j] : sf[q * 32];
            float x0 = f.x, x1 = f.x, y0 = f.y, y1 = f.y;
            for (int o = 16; o > 0; o >>= 1) {
                x0 = fminf(x0, __shfl_xor_sync(0xffffffffu, x0, o));
                x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o));
                y0 = fminf(y0, __shfl_xor_sync(0xffffffffu, y0, o));
                y1 = fmaxf(y1, __shfl_xor_sync(0xffffffffu, y1, o));
            }
            if (lane == 0) sbox[q] = make_float4(x0, x1, y0, y1);
        }
    }
    __syncthreads();
    // |d2_fp32 - d2_fp64| <= ~5e-7 * maxc^2 (rounding of the coordinates and of d2): margin 4x that
    const float maxc = __uint_as_float(smax) + 1.f;
    const float margin = 1.f + 2e-6f * maxc * maxc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k0 = (blockIdx.x * kNbrWarps + warp) * kNbrPerWarp;
    for (int k = k0; k < min(k0 + kNbrPerWarp, cs.c); ++k) {
        const double2 ck = sc[k];
        const float2 fk = sf[k];
        // pass 1 (fp32): the G-th smallest approximate d^2 over the 64 clusters around k
        // in curve order (Hilbert neighbours are spatial neighbours) -- an upper bound
        // of the true G-th smallest, so pass 2's filter still keeps every true candidate
        float fd[G];
#pragma unroll
        for (int r = 0; r < G; ++r) fd[r] = INFINITY;
        const int w0 = max(0, min(k - 32, cs.c - 64));
        for (int j = w0 + lane; j < min(w0 + 64, cs.c); j += 32) {
            const float2 fj = sf[j];
            const float dx = fj.x - fk.x, dy = fj.y - fk.y;
            float v = fmaf(dx, dx, dy * dy);
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const float lo = fminf(v, fd[r]);
                v = fmaxf(v, fd[r]);
                fd[r] = lo;
            }
        }
        // warp-wide G-th smallest: repeatedly extract the minimum
        float thr = INFINITY;
        {
            int head = 0;
#pragma unroll
            for (int r = 0; r < G; ++r) {
                float mine = fd[0];
#pragma unroll
                for (int q = 1; q < G; ++q) mine = q == head ? fd[q] : mine;
                if (head >= G) mine = INFINITY;
                float m = mine;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
                const unsigned who = __ballot_sync(0xffffffffu, mine == m && head < G);
                if (lane == __ffs(who) - 1) ++head;
                thr = m;
            }
        }
        thr = thr * 1.0001f + margin;
        // pass 2 (exact binary64) over the candidates under the threshold only
        double d[G];
        int jj[G];
#pragma unroll
        for (int r = 0; r < G; ++r) {
            d[r] = INFINITY;
            jj[r] = INT32_MAX;
        }
        // only the 32-cluster runs whose box comes within the threshold (a lower bound of the
        // fp32 distance to every member, with a relative margin) are scanned
        const float bthr = thr * (1.f + 1e-5f);
        for (int q0 = 0; q0 < nchunk; q0 += 32) {
            bool near = false;
            if (q0 + lane < nchunk) {
                const float4 bx = sbox[q0 + lane];
                const float ex = fmaxf(0.f, fmaxf(bx.x - fk.x, fk.x - bx.y));
                const float ey = fmaxf(0.f, fmaxf(bx.z - fk.y, fk.y - bx.w));
                near = ex * ex + ey * ey <= bthr;
            }
            for (unsigned m = __ballot_sync(0xffffffffu, near); m; m &= m - 1) {
                const int j = (q0 + __ffs(m) - 1) * 32 + lane;
                if (j >= cs.c) continue;
                const float2 fj = sf[j];
                const float fx = fj.x - fk.x, fy = fj.y - fk.y;
                if (fmaf(fx, fx, fy * fy) > thr) continue;
                const double2 cj = sc[j];
                const double dx = __dsub_rn(cj.x, ck.x), dy = __dsub_rn(cj.y, ck.y);
                const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                if (pair_lt(d2, j, d[G - 1], jj[G - 1])) topk_push<G>(d, jj, d2, j);
            }
        }
        double od[G];
        int oj[G];
        warp_topk<G>(d, jj, G, od, oj);
        if (lane == 0) {
            int32_t* sel = nbr_cl + (int64_t(b) * cs.c + k) * G;
            int ns = 0;
            sel[ns++] = k;
#pragma unroll
            for (int r = 0; r < G; ++r)
                if (ns < G && oj[r] != k) sel[ns++] = oj[r];
        }
    }
}

static int launch_nbr(const double2* cent, int64_t batch, const ClusterShape& cs, int32_t* nbr, cudaStream_t st) {
    const size_t smem = size_t(cs.c) * sizeof(double2) + size_t((cs.c + 1) & ~1) * sizeof(float2) +
                        size_t((cs.c + 31) / 32) * sizeof(float4);
    if (smem > 200 * 1024) return -1;  // very large images: the generic kernel
    const dim3 grid(unsigned((cs.c + kNbrWarps * kNbrPerWarp - 1) / (kNbrWarps * kNbrPerWarp)), unsigned(batch));
    switch (cs.g) {
#define AFFMAE_NBR(G_)                                                                                       \
    case G_: {                                                                                               \
        if (smem > 40 * 1024) /* + static shared memory must fit too */                                    \
            AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(nbr_v2_kernel<G_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                   int(smem)));                                              \
        nbr_v2_kernel<G_><<<grid, kNbrWarps * 32, smem, st>>>(cent, cs, nbr);                                \
        break;                                                                                               \
    }
        AFFMAE_NBR(1)
        AFFMAE_NBR(2)
        AFFMAE_NBR(3)
        AFFMAE_NBR(4)
        AFFMAE_NBR(5)
        AFFMAE_NBR(6)
        AFFMAE_NBR(7)
        AFFMAE_NBR(8)
#undef AFFMAE_NBR
        default:
            return -1;
    }
    AFFMAE_LAUNCH_CHECK("nbr_v2_kernel");
    return AFFMAE_OK;
}

// reverse-neighbour CSR: in-degree, per-image scan, fill, per-list sort
__global__ void indeg_kernel(const int32_t* __restrict__ nbr_cl, int64_t batch, ClusterShape cs,
                             int32_t* __restrict__ cnt) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * cs.c * cs.g) return;
    int64_t b = i / (int64_t(cs.c) * cs.g);
    atomicAdd(cnt + b * (cs.c + 1) + nbr_cl[i], 1);
}

__global__ void rev_scan_kernel(int32_t* __restrict__ cnt, ClusterShape cs) {
    // one CTA per image: exclusive scan of cnt[0..C] in place (cnt[C] = total)
    __shared__ int32_t part[1024];
    int32_t* c = cnt + int64_t(blockIdx.x) * (cs.c + 1);
    const int t = threadIdx.x, nt = blockDim.x, len = cs.c + 1;
    const int per = (len + nt - 1) / nt, b = t * per, e = min(len, b + per);
    int32_t s = 0;
    for (int i = b; i < e; ++i) s += c[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        int32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - s;
    for (int i = b; i < e; ++i) {
        int32_t v = c[i];
        c[i] = run;
        run += v;
    }
}

__global__ void rev_fill_kernel(const int32_t* __restrict__ nbr_cl, int64_t batch, ClusterShape cs,
                                const int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                                int32_t* __restrict__ rev_cl) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * cs.c * cs.g) return;
    const int64_t per = int64_t(cs.c) * cs.g;
    int64_t b = i / per;
    int k = int((i - b * per) / cs.g);
    int t = nbr_cl[i];
    int slot = atomicAdd(cursor + b * (cs.c + 1) + t, 1);
    rev_cl[b * per + off[b * (cs.c + 1) + t] + slot] = k;
}

__global__ void rev_sort_kernel(const int32_t* __restrict__ off, int64_t batch, ClusterShape cs,
                                int32_t* __restrict__ rev_cl) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * cs.c) return;
    int64_t b = i / cs.c;
    int c = int(i - b * cs.c);
    const int32_t* o = off + b * (cs.c + 1);
    int32_t* l = rev_cl + b * int64_t(cs.c) * cs.g;
    for (int x = o[c] + 1; x < o[c + 1]; ++x) {
        int v = l[x], y = x;
        while (y > o[c] && l[y - 1] > v) {
            l[y] = l[y - 1];
            --y;
        }
        l[y] = v;
    }
}

// Whole reverse CSR of one image in one CTA (shared-memory in-degree counts,
// scan, atomic fill, per-list insertion sort) -- the four kernels above fused
// for images whose counts fit in shared memory.
__global__ void __launch_bounds__(1024) rev_csr_kernel(const int32_t* __restrict__ nbr_cl, ClusterShape cs,
                                                       int32_t* __restrict__ rev_off, int32_t* __restrict__ rev_cl) {
    extern __shared__ int32_t rsm[];
    __shared__ int32_t part[1024];
    const int C = cs.c, t = threadIdx.x, nt = blockDim.x;
    int32_t* cnt = rsm;          // [C + 1] counts -> offsets
    int32_t* cur = rsm + C + 1;  // [C] fill cursors
    const int64_t per = int64_t(C) * cs.g;
    const int32_t* nb = nbr_cl + blockIdx.x * per;
    int32_t* off = rev_off + int64_t(blockIdx.x) * (C + 1);
    int32_t* rl = rev_cl + blockIdx.x * per;
    for (int i = t; i <= C; i += nt) cnt[i] = 0;
    __syncthreads();
    for (int64_t i = t; i < per; i += nt) atomicAdd(&cnt[nb[i]], 1);
    __syncthreads();
    const int len = C + 1, chunk = (len + nt - 1) / nt, b0 = t * chunk, e0 = min(len, b0 + chunk);
    int32_t sum = 0;
    for (int i = b0; i < e0; ++i) sum += cnt[i];
    part[t] = sum;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        const int32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - sum;
    for (int i = b0; i < e0; ++i) {
        const int32_t v = cnt[i];
        cnt[i] = run;
        off[i] = run;
        if (i < C) cur[i] = run;
        run += v;
    }
    __syncthreads();
    for (int64_t i = t; i < per; i += nt) rl[atomicAdd(&cur[nb[i]], 1)] = int(i / cs.g);
    __syncthreads();
    for (int c = t; c < C; c += nt) {  // ascending query clusters per list
        const int lo = cnt[c], hi = cnt[c + 1];
        for (int x = lo + 1; x < hi; ++x) {
            const int v = rl[x];
            int y = x;
            while (y > lo && rl[y - 1] > v) {
                rl[y] = rl[y - 1];
                --y;
            }
            rl[y] = v;
        }
    }
}

// ------------------------------------------------------ NeighborIndex expand
__global__ void expand_rows_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ nbr_cl,
                                   int64_t batch, ClusterShape cs, int32_t* __restrict__ idx,
                                   uint8_t* __restrict__ valid) {
    // one thread per (image, curve position, slot): the row of token perm[pos]
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int M = cs.width;
    if (i >= batch * cs.n * M) return;
    int64_t pp = i / M;
    int s = int(i - pp * M);
    int64_t b = pp / cs.n;
    int pos = int(pp - b * cs.n);
    int k = cs.cluster_at(pos);
    const int32_t* nb = nbr_cl + (b * cs.c + k) * cs.g;
    const int32_t* pm = perm + b * cs.n;
    int start = 0, key = 0, ok = 0;
    for (int g = 0; g < cs.g; ++g) {
        int cl = nb[g], len = cs.len(cl);
        if (s < start + len) {
            key = pm[cs.off(cl) + s - start];
            ok = 1;
            break;
        }
        start += len;
    }
    int64_t row = b * cs.n + pm[pos];
    idx[row * M + s] = key;
    valid[row * M + s] = uint8_t(ok);
}

// ----------------------------------------------------------------- knn
// one warp per query: per-lane sorted top-k over a strided key subset, then
// a warp merge; (d^2 binary64, j) order (proj/src/geometry.cpp:196-214)
constexpr int kKnnMax = 32;
__global__ void knn_kernel(const float* __restrict__ queries, const float* __restrict__ keys,
                           int64_t batch, int64_t nq, int64_t nk, int k, int32_t* __restrict__ idx,
                           uint8_t* __restrict__ valid) {
    const int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= batch * nq) return;
    int64_t b = w / nq;
    const float2 q = reinterpret_cast<const float2*>(queries)[w];
    const float2* kb = reinterpret_cast<const float2*>(keys) + b * nk;
    const int kept = int(k < nk ? k : nk);
    double d[kKnnMax];
    int jj[kKnnMax];
    for (int r = 0; r < kKnnMax; ++r) {
        d[r] = INFINITY;
        jj[r] = INT32_MAX;
    }
    for (int64_t j = lane; j < nk; j += 32) {
        float2 p = kb[j];
        double dx = __dsub_rn(double(p.x), double(q.x)), dy = __dsub_rn(double(p.y), double(q.y));
        double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        topk_insert<kKnnMax>(d, jj, kept, d2, int(j));
    }
    double od[kKnnMax];
    int oj[kKnnMax];
    warp_topk<kKnnMax>(d, jj, kept, od, oj);
    // every lane holds the merged list; lane s writes slot s (k <= 32)
    int jv = 0;
#pragma unroll
    for (int t = 0; t < kKnnMax; ++t)
        if (t == lane) jv = oj[t];
    if (lane < k) {
        idx[w * k + lane] = lane < kept ? jv : 0;
        valid[w * k + lane] = lane < kept ? 1 : 0;
    }
}

// fp32 pre-filter of the exact binary64 scan.  d2f = the squared distance in fp32 is within a
// relative 2^-21 of the binary64 d^2 the reference compares (exact float differences, three
// roundings of 2^-24 each), so a key with d2f > (1 + 2^-17) * (current K-th binary64 d^2)
// cannot enter the top-K: it is skipped without the binary64 arithmetic (the FP64 pipe is the
// scan's bottleneck).  Every key that survives takes the exact path, so the selection and
// its tie order are unchanged.
__device__ __forceinline__ float knn_d2f(float2 p, float2 q) {
    const float dx = __fsub_rn(p.x, q.x), dy = __fsub_rn(p.y, q.y);
    return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}
__device__ __forceinline__ float knn_prune_bound(double kth) {
    return kth < 1e37 ? __double2float_ru(kth * (1.0 + 0x1p-17)) : INFINITY;
}

// Few keys per image (<= 1024) and k <= 8: the image's keys staged once per block in shared
// memory as binary64, one query per thread scanning all of them with a register top-K --
// the same (d^2 binary64 without FMA, index) order as the reference's scan, no warp merge.
template <int K>
__global__ void __launch_bounds__(256) knn_smem_kernel(const float* __restrict__ queries, const float* __restrict__ keys,
                                                       int64_t nq, int64_t nk, int k, int32_t* __restrict__ idx,
                                                       uint8_t* __restrict__ valid) {
    extern __shared__ double2 skeys[];
    float2* fkeys = reinterpret_cast<float2*>(skeys + nk);
    const int64_t b = blockIdx.y;
    const float2* kb = reinterpret_cast<const float2*>(keys) + b * nk;
    for (int64_t j = threadIdx.x; j < nk; j += blockDim.x) {
        const float2 p = kb[j];
        skeys[j] = make_double2(double(p.x), double(p.y));
        fkeys[j] = p;
    }
    __syncthreads();
    const int64_t qi = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    const int64_t w = b * nq + qi;
    const float2 q = reinterpret_cast<const float2*>(queries)[w];
    const double qx = double(q.x), qy = double(q.y);
    const int kept = int(k < nk ? k : nk);
    double d[K];
    int jj[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
        d[r] = INFINITY;
        jj[r] = INT32_MAX;
    }
    // Prune bound before the scan: the K-th smallest fp32 d^2 over an evenly spaced sample of
    // 4K keys is >= the true K-th (a subset's K-th is never smaller), so keys beyond it (with
    // the knn_prune_bound margin) are skipped from the first key on -- the scan's register
    // insertions, and the warp divergence they cause, drop to the few keys inside it.
    float thr = INFINITY;
    // the scan starts at the sample nearest to the query and wraps around: with spatially
    // ordered keys (the model's token order) the K-th best tightens within the first keys, so
    // the pre-filter rejects nearly all the rest -- scanning from key 0 let the far keys of a
    // raster order through the filter and into the binary64 insertion (70 % of the kernel's
    // instructions).  The selection is by (d², j) and does not depend on the order.
    int start = 0;
    if (nk >= 8 * K) {
        float sd[K];
        float best = INFINITY;
#pragma unroll
        for (int r = 0; r < K; ++r) sd[r] = INFINITY;
        for (int i = 0; i < 4 * K; ++i) {
            const int si = int(int64_t(i) * nk / (4 * K));
            float v = knn_d2f(fkeys[si], q);
            if (v < best) {
                best = v;
                start = si;
            }
#pragma unroll
            for (int r = 0; r < K; ++r) {
                const float lo = fminf(v, sd[r]);
                v = fmaxf(v, sd[r]);
                sd[r] = lo;
            }
        }
        thr = sd[K - 1] < 1e37f ? __fmul_ru(sd[K - 1], 1.f + 0x1p-16f) : INFINITY;
    }
    for (int c = 0, j = start; c < int(nk); ++c, j = j + 1 < int(nk) ? j + 1 : 0) {
        const float2 pf = fkeys[j];
        if (knn_d2f(pf, q) > thr) continue;
        const double2 p = skeys[j];
        const double dx = __dsub_rn(p.x, qx), dy = __dsub_rn(p.y, qy);
        double nd = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        if (!pair_lt(nd, j, d[K - 1], jj[K - 1])) continue;  // (d², j) order: ties keep the lower index
        int nj = j;
#pragma unroll
        for (int r = 0; r < K; ++r) {  // register-resident sorted insertion by (d^2, j), K >= k
            if (pair_lt(nd, nj, d[r], jj[r])) {
                const double td = d[r];
                const int tj = jj[r];
                d[r] = nd;
                jj[r] = nj;
                nd = td;
                nj = tj;
            }
        }
        thr = fminf(thr, knn_prune_bound(d[K - 1]));
    }
#pragma unroll
    for (int t = 0; t < K; ++t)
        if (t < k) {
            idx[w * k + t] = t < kept ? jj[t] : 0;
            valid[w * k + t] = t < kept ? 1 : 0;
        }
}

// ---------------------------------------------- grid-accelerated exact knn
// Large key sets: the image's keys are bucketed once into a uniform grid of
// ~2 keys per cell (counting sort in global memory); each query (one thread)
// walks square rings of cells around its own, keeping a sorted top-K of
// (d^2 binary64, j), and stops once its K-th best d^2 is strictly below the
// squared distance to every unvisited cell (minus a rounding margin) -- the
// same selection as the brute-force scan, at O(K) candidates per query.
struct KnnGrid {
    double x0, y0, w;  // origin, cell side (square cells)
    int g;             // cells per side
    int pad;
};
__global__ void knn_grid_prm_kernel(const float* __restrict__ keys, int64_t nk, KnnGrid* __restrict__ prm) {
    __shared__ float red[4][32];
    const float2* kb = reinterpret_cast<const float2*>(keys) + int64_t(blockIdx.x) * nk;
    float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (int64_t i = threadIdx.x; i < nk; i += blockDim.x) {
        const float2 v = kb[i];
        x0 = fminf(x0, v.x); x1 = fmaxf(x1, v.x); y0 = fminf(y0, v.y); y1 = fmaxf(y1, v.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        x0 = fminf(x0, __shfl_xor_sync(0xffffffffu, x0, o)); x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o));
        y0 = fminf(y0, __shfl_xor_sync(0xffffffffu, y0, o)); y1 = fmaxf(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][warp] = x0; red[1][warp] = x1; red[2][warp] = y0; red[3][warp] = y1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            x0 = fminf(x0, red[0][w]); x1 = fmaxf(x1, red[1][w]); y0 = fminf(y0, red[2][w]); y1 = fmaxf(y1, red[3][w]);
        }
        KnnGrid p;
        p.g = max(1, min(1024, int(ceil(sqrt(double(nk) / 2.0)))));
        const double ext = fmax(double(x1) - double(x0), double(y1) - double(y0));
        p.w = ext > 0.0 ? ext / p.g * (1.0 + 1e-9) : 1.0;  // keys never land past the last cell
        p.x0 = double(x0);
        p.y0 = double(y0);
        p.pad = 0;
        prm[blockIdx.x] = p;
    }
}
__device__ __forceinline__ int knn_cell(double v, double v0, double w, int g) {
    return min(g - 1, max(0, int((v - v0) / w)));
}
__global__ void knn_grid_count_kernel(const float* __restrict__ keys, int64_t batch, int64_t nk,
                                      const KnnGrid* __restrict__ prm, int64_t cells_cap, int32_t* __restrict__ cnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * nk) return;
    const int64_t b = i / nk;
    const KnnGrid p = prm[b];
    const float2 v = reinterpret_cast<const float2*>(keys)[i];
    atomicAdd(cnt + b * cells_cap + knn_cell(v.y, p.y0, p.w, p.g) * p.g + knn_cell(v.x, p.x0, p.w, p.g), 1);
}
__global__ void knn_grid_scan_kernel(int32_t* __restrict__ cnt, int64_t cells_cap, int32_t* __restrict__ cur) {
    __shared__ int32_t part[1024];
    int32_t* c = cnt + int64_t(blockIdx.x) * cells_cap;
    int32_t* u = cur + int64_t(blockIdx.x) * cells_cap;
    const int t = threadIdx.x, nt = blockDim.x;
    const int64_t per = (cells_cap + nt - 1) / nt, b0 = t * per, e0 = min(cells_cap, b0 + per);
    int32_t s2 = 0;
    for (int64_t i = b0; i < e0; ++i) s2 += c[i];
    part[t] = s2;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        const int32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - s2;
    for (int64_t i = b0; i < e0; ++i) {
        const int32_t v = c[i];
        c[i] = run;
        u[i] = run;
        run += v;
    }
}
__global__ void knn_grid_fill_kernel(const float* __restrict__ keys, int64_t batch, int64_t nk,
                                     const KnnGrid* __restrict__ prm, int64_t cells_cap, int32_t* __restrict__ cur,
                                     int32_t* __restrict__ items, float2* __restrict__ item_xy) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * nk) return;
    const int64_t b = i / nk;
    const KnnGrid p = prm[b];
    const float2 v = reinterpret_cast<const float2*>(keys)[i];
    const int c = knn_cell(v.y, p.y0, p.w, p.g) * p.g + knn_cell(v.x, p.x0, p.w, p.g);
    const int pos = atomicAdd(cur + b * cells_cap + c, 1);
    items[b * nk + pos] = int32_t(i - b * nk);
    item_xy[b * nk + pos] = v;
}
template <int KM>
__global__ void __launch_bounds__(128) knn_grid_query_kernel(const float* __restrict__ queries, int64_t batch,
                                                             int64_t nq, int64_t nk, int k,
                                                             const KnnGrid* __restrict__ prm, int64_t cells_cap,
                                                             const int32_t* __restrict__ off,
                                                             const int32_t* __restrict__ items,
                                                             const float2* __restrict__ item_xy,
                                                             int32_t* __restrict__ idx, uint8_t* __restrict__ valid) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * nq) return;
    const int64_t b = i / nq;
    const KnnGrid p = prm[b];
    const int32_t* co = off + b * cells_cap;
    const int32_t* it = items + b * nk;
    const float2* ixy = item_xy + b * nk;
    const float2 q = reinterpret_cast<const float2*>(queries)[i];
    const double qx = q.x, qy = q.y;
    const int kept = int(k < nk ? k : nk);
    double d[KM];
    int jj[KM];
#pragma unroll
    for (int r = 0; r < KM; ++r) {
        d[r] = INFINITY;
        jj[r] = INT32_MAX;
    }
    float thr = INFINITY;  // fp32 pre-filter (knn_prune_bound)
    const int g = p.g;
    const int qcx = knn_cell(qx, p.x0, p.w, g), qcy = knn_cell(qy, p.y0, p.w, g);
    int found = 0;
    bool done = false;
    constexpr int kMaxRings = 24;  // far / clumped cases: exact scan of all keys instead
    for (int ring = 0; ring <= min(g, kMaxRings); ++ring) {
        const int x0 = qcx - ring, x1 = qcx + ring, y0 = qcy - ring, y1 = qcy + ring;
        // perimeter cells of the ring, row by row, as one flat loop (no lambda: the
        // top-K list must stay in registers)
        for (int cy = max(y0, 0); cy <= min(y1, g - 1); ++cy) {
            const bool edge = cy == y0 || cy == y1;
            const int ca = edge ? max(x0, 0) : x0, cb = edge ? min(x1, g - 1) : x1;
            const int step = edge ? 1 : max(1, x1 - x0);
            for (int cx = ca; cx <= cb; cx += step) {
                if (cx < 0 || cx > g - 1) continue;
                const int cell = cy * g + cx;
                const int t1 = co[cell + 1];
                for (int t = co[cell]; t < t1; ++t) {
                    const float2 v = ixy[t];
                    ++found;
                    if (knn_d2f(v, q) > thr) continue;
                    const int j = it[t];
                    const double dx = __dsub_rn(double(v.x), qx), dy = __dsub_rn(double(v.y), qy);
                    const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                    if (!pair_lt(d2, j, d[KM - 1], jj[KM - 1])) continue;
                    double nd = d2;
                    int nj = j;
#pragma unroll
                    for (int r = 0; r < KM; ++r) {
                        if (pair_lt(nd, nj, d[r], jj[r])) {
                            const double td = d[r];
                            const int tj = jj[r];
                            d[r] = nd;
                            jj[r] = nj;
                            nd = td;
                            nj = tj;
                        }
                    }
                    thr = knn_prune_bound(d[KM - 1]);
                }
            }
        }
        if (x0 <= 0 && y0 <= 0 && x1 >= g - 1 && y1 >= g - 1) {  // whole grid searched
            done = true;
            break;
        }
        if (found >= kept) {
            // distance from q to the outside of the searched (2 ring + 1)^2 block
            double lb = INFINITY;
            if (x0 > 0) lb = fmin(lb, qx - (p.x0 + x0 * p.w));
            if (x1 < g - 1) lb = fmin(lb, p.x0 + (x1 + 1) * p.w - qx);
            if (y0 > 0) lb = fmin(lb, qy - (p.y0 + y0 * p.w));
            if (y1 < g - 1) lb = fmin(lb, p.y0 + (y1 + 1) * p.w - qy);
            lb -= 1e-9 * p.w * g;
            double dk = INFINITY;
#pragma unroll
            for (int r = 0; r < KM; ++r)
                if (r == kept - 1) dk = d[r];
            if (lb > 0.0 && dk < lb * lb) {
                done = true;
                break;
            }
        }
    }
    if (!done) {  // ring budget exhausted: brute force over the image's keys (same order rule)
#pragma unroll
        for (int r = 0; r < KM; ++r) {
            d[r] = INFINITY;
            jj[r] = INT32_MAX;
        }
        for (int64_t t = 0; t < nk; ++t) {
            const float2 v = ixy[t];
            const int j = it[t];
            const double dx = __dsub_rn(double(v.x), qx), dy = __dsub_rn(double(v.y), qy);
            const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
            if (!pair_lt(d2, j, d[KM - 1], jj[KM - 1])) continue;
            double nd = d2;
            int nj = j;
#pragma unroll
            for (int r = 0; r < KM; ++r) {
                if (pair_lt(nd, nj, d[r], jj[r])) {
                    const double td = d[r];
                    const int tj = jj[r];
                    d[r] = nd;
                    jj[r] = nj;
                    nd = td;
                    nj = tj;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < KM; ++r)
        if (r < k) {
            idx[i * k + r] = r < kept ? jj[r] : 0;
            valid[i * k + r] = r < kept ? 1 : 0;
        }
}

// ================================================================= host
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct IndexWs {
    uint64_t* keys[2];
    uint32_t* vals[2];
    uint32_t* hist;
    unsigned long long* gaps;
    double2* cent;
    int32_t* cursor;
    float2* minmax;  // per (image, axis) {min, max} of the axis statistics pass
    int* hard;       // 1: some image needs the axis sort for its min_gap
    size_t bytes;
};

static IndexWs carve(int64_t batch, int64_t n, int64_t c, void* base) {
    IndexWs w{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    };
    const size_t e = size_t(batch) * n * 2;  // x and y segments
    w.keys[0] = reinterpret_cast<uint64_t*>(take(e * 8));
    w.keys[1] = reinterpret_cast<uint64_t*>(take(e * 8));
    w.vals[0] = reinterpret_cast<uint32_t*>(take(e * 4));
    w.vals[1] = reinterpret_cast<uint32_t*>(take(e * 4));
    w.hist = reinterpret_cast<uint32_t*>(take(radix_hist_elems(int64_t(e)) * 4));
    w.gaps = reinterpret_cast<unsigned long long*>(take(size_t(batch) * 2 * 8));
    w.cent = reinterpret_cast<double2*>(take(size_t(batch) * c * sizeof(double2)));
    w.cursor = reinterpret_cast<int32_t*>(take(size_t(batch) * (c + 1) * 4));
    w.minmax = reinterpret_cast<float2*>(take(size_t(batch) * 2 * sizeof(float2)));
    w.hard = reinterpret_cast<int*>(take(16));
    w.bytes = off;
    return w;
}

static unsigned blocks(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

// sfc_order for the batch; leaves the sorted token ids in *sorted_vals
static int sfc_core(const float* coords, int64_t batch, int64_t n, IndexWs& w, uint32_t** sorted_vals,
                    cudaStream_t st) {
    const int64_t e = batch * n * 2;
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.gaps, 0xFF, size_t(batch) * 2 * 8, st));
    // images of <= kSegSortMax tokens: min / max and min_gap from the bucket pass, the axis
    // sort only when a bucket holds two distinct values (device-side gate)
    const bool stats = n <= kSegSortMax;
    const int* gate = nullptr;
    if (stats) {
        AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.hard, 0, sizeof(int), st));
        axis_stats_kernel<<<unsigned(batch * 2), 1024, 0, st>>>(coords, n, w.minmax, w.gaps, w.hard);
        AFFMAE_LAUNCH_CHECK("axis_stats_kernel");
        gate = w.hard;
    }
    axis_keys_kernel<<<blocks(e), 256, 0, st>>>(coords, batch, n, w.keys[0], gate);
    AFFMAE_LAUNCH_CHECK("axis_keys_kernel");
    uint64_t* k = w.keys[0];
    uint32_t* v = nullptr;
    bool gaps_done = false;
    int rc = segmented_sort(k, v, w.keys[1], nullptr, batch * 2, n, 32 + bits_for(batch * 2), w.hist, st,
                            w.gaps, &gaps_done, gate);
    if (rc) return rc;
    if (!gaps_done) gap_kernel<<<blocks(e), 256, 0, st>>>(k, batch * 2, n, w.gaps);
    // the sorted axes live in w.keys[0] or w.keys[1]; the Hilbert keys go to the other buffer
    uint64_t* hk = k == w.keys[0] ? w.keys[1] : w.keys[0];
    hilbert_keys_kernel<<<blocks(batch * n), 256, 0, st>>>(coords, batch, n, k, stats ? w.minmax : nullptr, w.gaps,
                                                           hk, w.vals[0]);
    AFFMAE_LAUNCH_CHECK("hilbert_keys_kernel");
    k = hk;
    v = w.vals[0];
    rc = segmented_sort(k, v, hk == w.keys[0] ? w.keys[1] : w.keys[0], w.vals[1], batch, n, 32 + bits_for(batch),
                        w.hist, st);
    if (rc) return rc;
    *sorted_vals = v;
    return AFFMAE_OK;
}

size_t cluster_index_workspace(const affmae_cluster_geom* g) {
    if (!g || g->n_clusters <= 0) return 0;
    return carve(g->batch, g->tokens, g->n_clusters, nullptr).bytes;
}

int cluster_index_build(const affmae_cluster_geom* g, const float* coords, affmae_cluster_index* out,
                        void* workspace, size_t ws_bytes, void* stream) {
    if (!g || g->n_clusters <= 0) return fail(AFFMAE_ECONFIG, "cluster_index: geometry not derived");
    if (!coords || !out || !out->perm || !out->cluster_of || !out->nbr_cl || !out->rev_off || !out->rev_cl)
        return fail(AFFMAE_ECONFIG, "cluster_index: null pointer");
    if (g->groups_eff > kMaxGroups)
        return fail(AFFMAE_EUNSUPPORTED, "cluster_index: groups > 8 not compiled");
    if (g->tokens >= (int64_t(1) << 31)) return fail(AFFMAE_EUNSUPPORTED, "cluster_index: too many tokens");
    IndexWs w = carve(g->batch, g->tokens, g->n_clusters, workspace);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "cluster_index: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const ClusterShape cs = make_shape(*g);
    const int64_t B = g->batch, n = g->tokens;
    uint32_t* sv = nullptr;
    int rc = sfc_core(coords, B, n, w, &sv, st);
    if (rc) return rc;
    perm_centroid_kernel<<<blocks(B * cs.c), 256, 0, st>>>(sv, coords, B, cs, out->perm, out->cluster_of, w.cent);
    {
        const int rc = launch_nbr(w.cent, B, cs, out->nbr_cl, st);
        if (rc > 0) return rc;
        if (rc < 0) nbr_kernel<<<blocks(B * cs.c * 32), 256, 0, st>>>(w.cent, B, cs, out->nbr_cl);
    }
    AFFMAE_LAUNCH_CHECK("nbr_kernel");
    const size_t rsmem = size_t(2 * cs.c + 1) * 4;
    if (rsmem <= 48 * 1024) {
        rev_csr_kernel<<<unsigned(B), 1024, rsmem, st>>>(out->nbr_cl, cs, out->rev_off, out->rev_cl);
    } else {  // very large images: global-memory passes
        AFFMAE_CUDA_CHECK(cudaMemsetAsync(out->rev_off, 0, size_t(B) * (cs.c + 1) * 4, st));
        AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.cursor, 0, size_t(B) * (cs.c + 1) * 4, st));
        const int64_t pairs = B * cs.c * cs.g;
        indeg_kernel<<<blocks(pairs), 256, 0, st>>>(out->nbr_cl, B, cs, out->rev_off);
        rev_scan_kernel<<<unsigned(B), 1024, 0, st>>>(out->rev_off, cs);
        rev_fill_kernel<<<blocks(pairs), 256, 0, st>>>(out->nbr_cl, B, cs, out->rev_off, w.cursor, out->rev_cl);
        rev_sort_kernel<<<blocks(B * cs.c), 256, 0, st>>>(out->rev_off, B, cs, out->rev_cl);
    }
    AFFMAE_LAUNCH_CHECK("reverse CSR");
    return AFFMAE_OK;
}

size_t sfc_order_workspace(int64_t batch, int64_t tokens) {
    if (batch < 0 || tokens < 1) return 0;
    return carve(batch, tokens, 1, nullptr).bytes;
}

int sfc_order(const float* coords, int64_t batch, int64_t n, int32_t* perm, void* workspace,
              size_t ws_bytes, void* stream) {
    if (n < 1) return fail(AFFMAE_ECONFIG, "sfc_order: empty point set");
    if (!coords || !perm) return fail(AFFMAE_ECONFIG, "sfc_order: null pointer");
    IndexWs w = carve(batch, n, 1, workspace);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "sfc_order: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    uint32_t* sv = nullptr;
    int rc = sfc_core(coords, batch, n, w, &sv, st);
    if (rc) return rc;
    ClusterShape cs{};
    cs.n = int32_t(n);
    cs.c = 1;
    cs.base = int32_t(n);
    perm_kernel<<<blocks(batch * n), 256, 0, st>>>(sv, batch, cs, perm, nullptr);
    AFFMAE_LAUNCH_CHECK("perm_kernel");
    return AFFMAE_OK;
}

int neighbor_expand(const affmae_cluster_geom* g, const int32_t* perm, const int32_t* nbr_cl,
                    int32_t* idx, uint8_t* valid, void* stream) {
    if (!g || g->n_clusters <= 0) return fail(AFFMAE_ECONFIG, "neighbor_expand: geometry not derived");
    if (!perm || !nbr_cl || !idx || !valid) return fail(AFFMAE_ECONFIG, "neighbor_expand: null pointer");
    const ClusterShape cs = make_shape(*g);
    const int64_t total = g->batch * g->tokens * g->width;
    if (total == 0) return AFFMAE_OK;
    expand_rows_kernel<<<blocks(total), 256, 0, as_stream(stream)>>>(perm, nbr_cl, g->batch, cs, idx, valid);
    AFFMAE_LAUNCH_CHECK("expand_rows_kernel");
    return AFFMAE_OK;
}

int knn(const float* queries, const float* keys, int64_t batch, int64_t nq, int64_t nk, int64_t k,
        int32_t* idx, uint8_t* valid, void* stream) {
    if (nk < 1) return fail(AFFMAE_ECONFIG, "knn: empty key set");
    if (k < 1) return fail(AFFMAE_ECONFIG, "knn: k must be >= 1");
    if (k > kKnnMax) return fail(AFFMAE_EUNSUPPORTED, "knn: k > 32 not compiled");
    if (!queries || !keys || !idx || !valid) return fail(AFFMAE_ECONFIG, "knn: null pointer");
    if (batch * nq == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    if (k <= 8 && nk <= 1024 && nq >= 256) {  // few keys, many queries: keys in shared memory
        const dim3 grid(unsigned((nq + 255) / 256), unsigned(batch));
        const size_t smem = size_t(nk) * (sizeof(double2) + sizeof(float2));
        if (smem > 40 * 1024)
            AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(knn_smem_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(smem)));
        knn_smem_kernel<8><<<grid, 256, smem, st>>>(queries, keys, nq, nk, int(k), idx, valid);
        AFFMAE_LAUNCH_CHECK("knn_smem_kernel");
        return AFFMAE_OK;
    }
    if (nk < 512 || nq * nk < (int64_t(1) << 20)) {  // small problems: brute force
        knn_kernel<<<blocks(batch * nq * 32), 256, 0, st>>>(queries, keys, batch, nq, nk, int(k), idx, valid);
        AFFMAE_LAUNCH_CHECK("knn_kernel");
        return AFFMAE_OK;
    }
    // grid state from the stream-ordered allocator (capturable; freed on the stream)
    const int gmax = max(1, min(1024, int(std::ceil(std::sqrt(double(nk) / 2.0)))));
    const int64_t cells_cap = int64_t(gmax) * gmax + 1;
    const size_t bytes = align256(size_t(batch) * sizeof(KnnGrid)) + 2 * align256(size_t(batch) * cells_cap * 4) +
                         align256(size_t(batch) * nk * 4) + align256(size_t(batch) * nk * 8);
    uint8_t* base = nullptr;
    AFFMAE_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&base), bytes, st));
    uint8_t* q = base;
    auto take = [&](size_t n) {
        uint8_t* r = q;
        q += align256(n);
        return r;
    };
    auto* prm = reinterpret_cast<KnnGrid*>(take(size_t(batch) * sizeof(KnnGrid)));
    auto* cnt = reinterpret_cast<int32_t*>(take(size_t(batch) * cells_cap * 4));
    auto* cur = reinterpret_cast<int32_t*>(take(size_t(batch) * cells_cap * 4));
    auto* items = reinterpret_cast<int32_t*>(take(size_t(batch) * nk * 4));
    auto* ixy = reinterpret_cast<float2*>(take(size_t(batch) * nk * 8));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(cnt, 0, size_t(batch) * cells_cap * 4, st));
    knn_grid_prm_kernel<<<unsigned(batch), 256, 0, st>>>(keys, nk, prm);
    knn_grid_count_kernel<<<blocks(batch * nk), 256, 0, st>>>(keys, batch, nk, prm, cells_cap, cnt);
    knn_grid_scan_kernel<<<unsigned(batch), 1024, 0, st>>>(cnt, cells_cap, cur);
    knn_grid_fill_kernel<<<blocks(batch * nk), 256, 0, st>>>(keys, batch, nk, prm, cells_cap, cur, items, ixy);
    const unsigned nb = unsigned((batch * nq + 127) / 128);
    if (k <= 8)
        knn_grid_query_kernel<8><<<nb, 128, 0, st>>>(queries, batch, nq, nk, int(k), prm, cells_cap, cnt, items, ixy,
                                                      idx, valid);
    else if (k <= 16)
        knn_grid_query_kernel<16><<<nb, 128, 0, st>>>(queries, batch, nq, nk, int(k), prm, cells_cap, cnt, items,
                                                       ixy, idx, valid);
    else
        knn_grid_query_kernel<32><<<nb, 128, 0, st>>>(queries, batch, nq, nk, int(k), prm, cells_cap, cnt, items,
                                                       ixy, idx, valid);
    AFFMAE_LAUNCH_CHECK("knn_grid");
    AFFMAE_CUDA_CHECK(cudaFreeAsync(base, st));
    return AFFMAE_OK;
}

}  // namespace affmae_b200
