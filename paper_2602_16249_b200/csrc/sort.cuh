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

// ----------------------------------------------------- segmented CTA sort
// Segments of <= kSegSortMax keys (one image's tokens) sort inside one CTA's
// shared memory: stable LSD passes over the LOW 32 bits of the keys, only for
// the key bytes that vary within the segment (OR ^ AND of the keys), values =
// segment-local indices (every call site sorts (key, local index) pairs).
// Each of the 16 warps owns a contiguous element range walked in rounds of
// 32 in element order, so the per-(warp, digit) offsets give a stable order.
constexpr int kSegSortMax = 16384;
constexpr int kSegWarps = 32;

template <bool WRITE_VALS>
__global__ void __launch_bounds__(kSegWarps * 32) seg_sort_kernel(const uint64_t* __restrict__ kin, int64_t seglen,
                                                                  uint64_t* __restrict__ kout,
                                                                  uint32_t* __restrict__ vout) {
    extern __shared__ __align__(16) uint8_t sraw[];
    const int L = int(seglen);
    const int Lp = (L + 31) & ~31;
    uint32_t* ka = reinterpret_cast<uint32_t*>(sraw);
    uint32_t* kb = ka + Lp;
    uint16_t* va = reinterpret_cast<uint16_t*>(kb + Lp);
    uint16_t* vb = va + Lp;
    uint32_t* off = reinterpret_cast<uint32_t*>(vb + Lp);  // [kSegWarps][256]
    __shared__ uint32_t tot[256];
    __shared__ uint32_t red[2][kSegWarps];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint64_t* src = kin + int64_t(blockIdx.x) * seglen;
    uint32_t o = 0, a = 0xffffffffu;
    constexpr int U = 8;  // loads in flight per thread
    for (int i0 = t; i0 < L; i0 += U * kSegWarps * 32) {
        uint32_t k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kSegWarps * 32;
            k[u] = i < L ? uint32_t(__ldg(src + i)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kSegWarps * 32;
            if (i < L) {
                ka[i] = k[u];
                va[i] = uint16_t(i);
                o |= k[u];
                a &= k[u];
            }
        }
    }
    o = __reduce_or_sync(0xffffffffu, o);
    a = __reduce_and_sync(0xffffffffu, a);
    if (lane == 0) {
        red[0][warp] = o;
        red[1][warp] = a;
    }
    __syncthreads();
    uint32_t vary = 0;
    {
        uint32_t oo = 0, aa = 0xffffffffu;
        for (int w = 0; w < kSegWarps; ++w) {
            oo |= red[0][w];
            aa &= red[1][w];
        }
        vary = oo ^ aa;
    }
    const int per = ((Lp / 32 + kSegWarps - 1) / kSegWarps) * 32;  // elements per warp (multiple of 32)
    const int w0 = warp * per, w1 = min(w0 + per, L);
    for (int shift = 0; shift < 32; shift += 8) {
        if (((vary >> shift) & 0xFFu) == 0) continue;  // uniform across the CTA
        for (int i = t; i < kSegWarps * 256; i += blockDim.x) off[i] = 0;
        __syncthreads();
        // 1. per-warp digit counts
        for (int b = w0; b < w1 + 0; b += 32) {
            const int i = b + lane;
            const int d = i < w1 ? int((ka[i] >> shift) & 0xFF) : 256;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256 && __popc(peers & lt) == 0) off[warp * 256 + d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // 2. offsets in (digit, warp) order
        if (t < 256) {
            uint32_t s = 0;
            for (int w = 0; w < kSegWarps; ++w) {
                const uint32_t c = off[w * 256 + t];
                off[w * 256 + t] = s;
                s += c;
            }
            tot[t] = s;
        }
        __syncthreads();
        if (t < 32) {  // exclusive scan of the 256 digit totals by one warp
            uint32_t v[8], run = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                v[j] = tot[t * 8 + j];
                run += v[j];
            }
            uint32_t inc = run;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
                if (t >= d) inc += y;
            }
            uint32_t base = inc - run;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                tot[t * 8 + j] = base;
                base += v[j];
            }
        }
        __syncthreads();
        for (int i = t; i < kSegWarps * 256; i += blockDim.x) off[i] += tot[i & 255];
        __syncthreads();
        // 3. stable scatter
        for (int b = w0; b < w1; b += 32) {
            const int i = b + lane;
            const bool ok = i < w1;
            const uint32_t k = ok ? ka[i] : 0u;
            const int d = ok ? int((k >> shift) & 0xFF) : 256;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            uint32_t base = 0;
            if (ok) base = off[warp * 256 + d];
            __syncwarp();
            if (ok) {
                const uint32_t pos = base + __popc(peers & lt);
                kb[pos] = k;
                vb[pos] = va[i];
                if (__popc(peers & lt) == 0) off[warp * 256 + d] = base + __popc(peers);
            }
            __syncwarp();
        }
        __syncthreads();
        uint32_t* tk = ka;
        ka = kb;
        kb = tk;
        uint16_t* tv = va;
        va = vb;
        vb = tv;
    }
    const uint64_t hi = src[0] & 0xffffffff00000000ull;
    uint64_t* dk = kout + int64_t(blockIdx.x) * seglen;
    for (int i = t; i < L; i += blockDim.x) {
        dk[i] = hi | ka[i];
        if (WRITE_VALS) vout[int64_t(blockIdx.x) * seglen + i] = va[i];
    }
}

inline size_t seg_sort_smem(int64_t seglen) {
    const int64_t Lp = (seglen + 31) & ~int64_t(31);
    return size_t(Lp) * (4 + 4 + 2 + 2) + size_t(kSegWarps) * 256 * 4;
}

// Sorts nseg contiguous segments of seglen keys (key = seg << 32 | low 32 bits,
// values = segment-local indices) stably by the low bits.  On return
// keys/vals point at the sorted data (vals only if non-null).
inline int segmented_sort(uint64_t*& keys, uint32_t*& vals, uint64_t* keys_alt, uint32_t* vals_alt,
                          int64_t nseg, int64_t seglen, int end_bit, uint32_t* hist, cudaStream_t st) {
    if (nseg <= 0 || seglen <= 0) return AFFMAE_OK;
    if (seglen > kSegSortMax || seglen > 65536)
        return radix_sort(keys, vals, keys_alt, vals_alt, nseg * seglen, end_bit, hist, st);
    const size_t smem = seg_sort_smem(seglen);
    if (vals) {
        static bool attr = false;
        if (!attr) {
            AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(seg_sort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(seg_sort_smem(kSegSortMax))));
            attr = true;
        }
        seg_sort_kernel<true><<<unsigned(nseg), kSegWarps * 32, smem, st>>>(keys, seglen, keys_alt, vals_alt);
    } else {
        static bool attr = false;
        if (!attr) {
            AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(seg_sort_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(seg_sort_smem(kSegSortMax))));
            attr = true;
        }
        seg_sort_kernel<false><<<unsigned(nseg), kSegWarps * 32, smem, st>>>(keys, seglen, keys_alt, nullptr);
    }
    AFFMAE_LAUNCH_CHECK("seg_sort_kernel");
    uint64_t* tk = keys;
    keys = keys_alt;
    keys_alt = tk;
    if (vals) {
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
