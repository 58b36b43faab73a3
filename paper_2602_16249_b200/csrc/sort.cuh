// Stable LSD radix sort of (uint64 key, uint32 value) pairs, hand-written for
// the index builder and the merge selection.  Batched problems sort a
// composite key (segment << 32 | key32), so one global sort serves all images
// and stability keeps the reference's "ties by index" rule (std::stable_sort,
// proj/src/geometry.cpp:103-104; proj/src/merging.cpp:62-66).
//
// One pass = 8 key bits, three kernels:
//   upsweep   per 2048-element tile, 256-bin digit histogram -> hist[bin][tile]
//   scan      exclusive scan of hist in (bin, tile) order (single CTA)
//   downsweep per tile, stable local ranks (warp __match_any + per-warp digit
//             counts, processed in element order) -> scatter
#pragma once
#include "common.cuh"

namespace affmae_b200 {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 8;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 2048

static __global__ void radix_upsweep(const uint64_t* __restrict__ keys, int64_t n, int shift, int tiles,
                              uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kSortTile;
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        int64_t i = base + r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    hist[int64_t(threadIdx.x) * tiles + blockIdx.x] = h[threadIdx.x];
}

// per-bin exclusive scan over tiles (one CTA per digit bin); the bin total
// goes to tot[bin].  hist is [bin][tile].
static __global__ void radix_scan_bins(uint32_t* __restrict__ hist, int tiles, uint32_t* __restrict__ tot) {
    __shared__ uint32_t part[256];
    uint32_t* h = hist + int64_t(blockIdx.x) * tiles;
    const int t = threadIdx.x, nt = blockDim.x;
    const int per = (tiles + nt - 1) / nt, b = t * per, e = (b + per < tiles) ? b + per : tiles;
    uint32_t s = 0;
    for (int i = b; i < e; ++i) s += h[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        uint32_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t run = part[t] - s;
    for (int i = b; i < e; ++i) {
        uint32_t v = h[i];
        h[i] = run;
        run += v;
    }
    if (t == nt - 1) tot[blockIdx.x] = part[t];
}

template <bool HAS_VAL>
__global__ void radix_downsweep(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                int64_t n, int shift, int tiles, const uint32_t* __restrict__ offs,
                                const uint32_t* __restrict__ tot) {
    __shared__ uint32_t wcnt[kSortThreads / 32][257];
    __shared__ uint32_t run[256];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const unsigned lt = (1u << lane) - 1u;
    {   // exclusive scan of the 256 bin totals (every CTA recomputes it: 256 values)
        uint32_t v = tot[t];
        run[t] = v;
        __syncthreads();
        for (int o = 1; o < 256; o <<= 1) {
            uint32_t x = t >= o ? run[t - o] : 0;
            __syncthreads();
            run[t] += x;
            __syncthreads();
        }
        const uint32_t base = run[t] - v;
        __syncthreads();
        run[t] = base + offs[int64_t(t) * tiles + blockIdx.x];
    }
    const int64_t base = int64_t(blockIdx.x) * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        for (int i = t; i < (kSortThreads / 32) * 257; i += kSortThreads) (&wcnt[0][0])[i] = 0;
        __syncthreads();
        const int64_t i = base + r * kSortThreads + t;
        const bool ok = i < n;
        uint64_t k = 0;
        uint32_t v = 0;
        int d = 256;
        if (ok) {
            k = kin[i];
            if (HAS_VAL) v = vin[i];
            d = int((k >> shift) & 0xFF);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        if (rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (ok) {
            uint32_t pos = run[d] + rank;
            for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
            kout[pos] = k;
            if (HAS_VAL) vout[pos] = v;
        }
        __syncthreads();
        {
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kSortThreads / 32; ++w) tot += wcnt[w][t];
            run[t] += tot;
        }
        __syncthreads();
    }
}

inline size_t radix_hist_elems(int64_t n) {
    int64_t tiles = (n + kSortTile - 1) / kSortTile;
    return size_t(256) * size_t(tiles > 0 ? tiles : 1) + 256;  // + bin totals
}

// Sorts keys[0..n) (with vals if non-null) on bits [0, end_bit), ping-ponging
// with the alt buffers.  On return `keys`/`vals` point at the sorted data.
inline int radix_sort(uint64_t*& keys, uint32_t*& vals, uint64_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int end_bit, uint32_t* hist, cudaStream_t st) {
    if (n <= 0) return AFFMAE_OK;
    const int tiles = int((n + kSortTile - 1) / kSortTile);
    for (int shift = 0; shift < end_bit; shift += 8) {
        uint32_t* tot = hist + size_t(256) * tiles;
        radix_upsweep<<<tiles, kSortThreads, 0, st>>>(keys, n, shift, tiles, hist);
        radix_scan_bins<<<256, 256, 0, st>>>(hist, tiles, tot);
        if (vals)
            radix_downsweep<true><<<tiles, kSortThreads, 0, st>>>(keys, vals, keys_alt, vals_alt, n,
                                                                shift, tiles, hist, tot);
        else
            radix_downsweep<false><<<tiles, kSortThreads, 0, st>>>(keys, nullptr, keys_alt, nullptr,
                                                                 n, shift, tiles, hist, tot);
        AFFMAE_LAUNCH_CHECK("radix sort pass");
        uint64_t* tk = keys;
        keys = keys_alt;
        keys_alt = tk;
        uint32_t* tv = vals;
        vals = vals_alt;
        vals_alt = tv;
    }
    return AFFMAE_OK;
}

inline int bits_for(int64_t v) {
    int b = 0;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

// order-preserving float -> uint32 map (ascending)
__device__ __forceinline__ uint32_t float_order(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

}  // namespace affmae_b200
