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

// inverse of float_order
__device__ __forceinline__ float float_unorder(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// order-preserving float -> uint32 map (ascending)
__device__ __forceinline__ uint32_t float_order(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

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

// ----------------------------------------------------- segmented sort
// Segments of <= kSegSortMax keys (one image's tokens) sort in shared memory:
// stable LSD passes over the LOW 32 bits of the keys, only for the key bytes
// that vary within the segment (OR ^ AND of the keys), values = segment-local
// indices (every call site sorts (key, local index) pairs).  Each warp owns a
// contiguous element range walked in rounds of 32 in element order, so the
// per-(warp, digit) offsets give a stable order.
constexpr int kSegSortMax = 16384;
constexpr int kSegWarps = 16;

// One segment is spread over a thread-block
// cluster of CL CTAs (distributed shared memory): CTA r holds slice
// [r*S, (r+1)*S) of the segment.  Per 8-bit pass every CTA counts its digits
// per warp, publishes its digit totals, reads the other CTAs' totals over
// DSMEM to place its (digit, rank, warp) runs, and scatters keys straight into
// the owning CTA's next-pass buffer (st.shared::cluster).  Order is
// (digit, CTA rank, warp, element) -> stable.  With 32-64 segments (one per
// image or axis) this puts 128-256 CTAs on the 148 SMs instead of 32-64.
template <int CL>
struct SegClusterSmem {
    uint32_t ctot[256];   // this CTA's per-digit totals (read by the cluster)
    uint32_t tot[256];
    uint32_t red[2][kSegWarps];
    uint32_t vary[2];     // this CTA's OR / AND of its keys (read by the cluster)
};
inline int seg_slice(int64_t seglen, int cl) { return int((seglen + cl - 1) / cl); }
inline size_t seg_sort_cl_smem(int64_t seglen, int cl) {
    const int64_t Sp = (seg_slice(seglen, cl) + 31) & ~31;
    return size_t(Sp) * (4 + 4 + 2 + 2) + size_t(kSegWarps) * 256 * 4;
}

__device__ __forceinline__ uint32_t dsmem_map(const void* p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t dsmem_ld32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void dsmem_st32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared::cluster.u16 [%0], %1;\n" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ int cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return int(r);
}

// `gap_out` (optional, pre-set to ~0): per segment, the smallest positive
// difference of consecutive sorted keys read as float_order'ed floats
// (min_gap, proj/src/geometry.cpp:57-65), as binary64 bits.
template <bool WRITE_VALS, int CL>
__global__ void __launch_bounds__(kSegWarps * 32) seg_sort_cl_kernel(const uint64_t* __restrict__ kin,
                                                                     int64_t seglen, uint64_t* __restrict__ kout,
                                                                     uint32_t* __restrict__ vout,
                                                                     unsigned long long* __restrict__ gap_out,
                                                                     const int* __restrict__ run_flag) {
    // a device-side gate (graph-capturable): every CTA of the cluster reads the same flag and
    // leaves before the first cluster barrier
    if (run_flag && *run_flag == 0) return;
    extern __shared__ __align__(16) uint8_t sraw[];
    __shared__ SegClusterSmem<CL> cs;
    const int rank = cluster_rank();
    const int64_t seg = blockIdx.x / CL;
    const int L = int(seglen), S = (L + CL - 1) / CL;
    const int s0 = min(rank * S, L), n = min(s0 + S, L) - s0;
    const int Sp = (S + 31) & ~31;
    uint32_t* ka = reinterpret_cast<uint32_t*>(sraw);
    uint32_t* kb = ka + Sp;
    uint16_t* va = reinterpret_cast<uint16_t*>(kb + Sp);
    uint16_t* vb = va + Sp;
    uint32_t* off = reinterpret_cast<uint32_t*>(vb + Sp);  // [kSegWarps][256]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint64_t* src = kin + seg * seglen + s0;
    uint32_t o = 0, a = 0xffffffffu;
    constexpr int U = 4;
    for (int i0 = t; i0 < n; i0 += U * kSegWarps * 32) {
        uint32_t k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kSegWarps * 32;
            k[u] = i < n ? uint32_t(__ldg(src + i)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kSegWarps * 32;
            if (i < n) {
                ka[i] = k[u];
                va[i] = uint16_t(s0 + i);
                o |= k[u];
                a &= k[u];
            }
        }
    }
    o = __reduce_or_sync(0xffffffffu, o);
    a = __reduce_and_sync(0xffffffffu, a);
    if (lane == 0) {
        cs.red[0][warp] = o;
        cs.red[1][warp] = a;
    }
    __syncthreads();
    if (t == 0) {
        uint32_t oo = 0, aa = 0xffffffffu;
        for (int w = 0; w < kSegWarps; ++w) {
            oo |= cs.red[0][w];
            aa &= cs.red[1][w];
        }
        cs.vary[0] = oo;
        cs.vary[1] = aa;
    }
    cluster_sync_all();
    uint32_t vary;
    {
        uint32_t oo = 0, aa = 0xffffffffu;
#pragma unroll
        for (int r = 0; r < CL; ++r) {
            oo |= dsmem_ld32(dsmem_map(&cs.vary[0], r));
            aa &= dsmem_ld32(dsmem_map(&cs.vary[1], r));
        }
        vary = oo ^ aa;
    }
    // no CTA may leave (or rewrite) while a peer still reads its shared memory:
    // with constant keys no pass (and no later cluster barrier) follows
    cluster_sync_all();
    const int per = ((Sp / 32 + kSegWarps - 1) / kSegWarps) * 32;
    const int w0 = warp * per, w1 = min(w0 + per, n);
    for (int shift = 0; shift < 32; shift += 8) {
        if (((vary >> shift) & 0xFFu) == 0) continue;  // uniform across the cluster
        for (int i = t; i < kSegWarps * 256; i += blockDim.x) off[i] = 0;
        __syncthreads();
        for (int b = w0; b < w1; b += 32) {
            const int i = b + lane;
            const int d = i < w1 ? int((ka[i] >> shift) & 0xFF) : 256;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256 && __popc(peers & lt) == 0) off[warp * 256 + d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        if (t < 256) {
            uint32_t s = 0;
            for (int w = 0; w < kSegWarps; ++w) {
                const uint32_t c = off[w * 256 + t];
                off[w * 256 + t] = s;
                s += c;
            }
            cs.ctot[t] = s;
        }
        cluster_sync_all();  // every CTA's digit totals published
        uint32_t before = 0;
        if (t < 256) {
            uint32_t all = 0;
#pragma unroll
            for (int r = 0; r < CL; ++r) {
                const uint32_t v = r == rank ? cs.ctot[t] : dsmem_ld32(dsmem_map(&cs.ctot[t], r));
                all += v;
                before += r < rank ? v : 0u;
            }
            cs.tot[t] = all;
        }
        __syncthreads();
        if (t < 32) {  // exclusive scan of the 256 cluster-wide digit totals
            uint32_t v[8], run = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                v[j] = cs.tot[t * 8 + j];
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
                cs.tot[t * 8 + j] = base;
                base += v[j];
            }
        }
        __syncthreads();
        if (t < 256) cs.tot[t] += before;
        __syncthreads();
        for (int i = t; i < kSegWarps * 256; i += blockDim.x) off[i] += cs.tot[i & 255];
        __syncthreads();
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
                const int dr = int(pos / uint32_t(S)), dl = int(pos - uint32_t(dr) * uint32_t(S));
                dsmem_st32(dsmem_map(kb + dl, dr), k);
                dsmem_st16(dsmem_map(vb + dl, dr), va[i]);
                if (__popc(peers & lt) == 0) off[warp * 256 + d] = base + __popc(peers);
            }
            __syncwarp();
        }
        cluster_sync_all();  // all scatters landed; ctot may be rewritten
        uint32_t* tk = ka;
        ka = kb;
        kb = tk;
        uint16_t* tv = va;
        va = vb;
        vb = tv;
    }
    if (gap_out) {
        // the previous slice's last key (DSMEM) closes the gap across the slice boundary
        const uint32_t prev = (CL > 1 && rank > 0 && n > 0) ? dsmem_ld32(dsmem_map(ka + (S - 1), rank - 1)) : 0u;
        unsigned long long best = ~0ull;
        for (int i = t; i < n; i += blockDim.x) {
            if (s0 + i == 0) continue;
            const double a = double(float_unorder(i > 0 ? ka[i - 1] : prev)), b = double(float_unorder(ka[i]));
            const double d = __dsub_rn(b, a);
            if (d > 0.0) best = min(best, (unsigned long long)__double_as_longlong(d));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0 && best != ~0ull) atomicMin(gap_out + seg, best);
        if (CL > 1) cluster_sync_all();  // peers have read our last key
    }
    const uint64_t hi = kin[seg * seglen] & 0xffffffff00000000ull;
    uint64_t* dk = kout + seg * seglen + s0;
    for (int i = t; i < n; i += blockDim.x) {
        dk[i] = hi | ka[i];
        if (WRITE_VALS) vout[seg * seglen + s0 + i] = va[i];
    }
}

template <bool WRITE_VALS, int CL>
inline int launch_seg_sort_cl(const uint64_t* kin, int64_t nseg, int64_t seglen, uint64_t* kout, uint32_t* vout,
                              unsigned long long* gap_out, cudaStream_t st, const int* run_flag) {
    auto kern = seg_sort_cl_kernel<WRITE_VALS, CL>;
    const size_t smem = seg_sort_cl_smem(seglen, CL);
    // per call (cheap, and right for whichever device is current)
    AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(seg_sort_cl_smem(kSegSortMax, 1))));
    AFFMAE_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(nseg * CL));
    cfg.blockDim = dim3(kSegWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    AFFMAE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, kin, seglen, kout, vout, gap_out, run_flag));
    return AFFMAE_OK;
}

// CTAs per segment: at most one wave of CTAs on the SMs, slices >= 1024 keys.
inline int seg_cluster_size(int64_t nseg, int64_t seglen) {
    int cl = 1;
    while (cl < 8 && nseg * cl * 2 <= 2 * kNumSMs && seglen / (cl * 2) >= 1024) cl *= 2;
    return cl;
}

template <bool WRITE_VALS>
inline int launch_seg_sort(const uint64_t* kin, int64_t nseg, int64_t seglen, uint64_t* kout, uint32_t* vout,
                           unsigned long long* gap_out, cudaStream_t st, const int* run_flag) {
    switch (seg_cluster_size(nseg, seglen)) {
        case 8: return launch_seg_sort_cl<WRITE_VALS, 8>(kin, nseg, seglen, kout, vout, gap_out, st, run_flag);
        case 4: return launch_seg_sort_cl<WRITE_VALS, 4>(kin, nseg, seglen, kout, vout, gap_out, st, run_flag);
        case 2: return launch_seg_sort_cl<WRITE_VALS, 2>(kin, nseg, seglen, kout, vout, gap_out, st, run_flag);
        default: return launch_seg_sort_cl<WRITE_VALS, 1>(kin, nseg, seglen, kout, vout, gap_out, st, run_flag);
    }
}


// Sorts nseg contiguous segments of seglen keys (key = seg << 32 | low 32 bits,
// values = segment-local indices) stably by the low bits.  On return
// keys/vals point at the sorted data (vals only if non-null).  With `gap_out`
// the shared-memory path also writes the per-segment min_gap and sets
// *gaps_done; the global fallback leaves that to the caller.
// `run_flag` (shared-memory path only): a device int; the sort is skipped when it reads 0.
inline int segmented_sort(uint64_t*& keys, uint32_t*& vals, uint64_t* keys_alt, uint32_t* vals_alt,
                          int64_t nseg, int64_t seglen, int end_bit, uint32_t* hist, cudaStream_t st,
                          unsigned long long* gap_out = nullptr, bool* gaps_done = nullptr,
                          const int* run_flag = nullptr) {
    if (gaps_done) *gaps_done = false;
    if (nseg <= 0 || seglen <= 0) return AFFMAE_OK;
    if (seglen > kSegSortMax || seglen > 65536)
        return radix_sort(keys, vals, keys_alt, vals_alt, nseg * seglen, end_bit, hist, st);
    const int rc = vals ? launch_seg_sort<true>(keys, nseg, seglen, keys_alt, vals_alt, gap_out, st, run_flag)
                        : launch_seg_sort<false>(keys, nseg, seglen, keys_alt, nullptr, gap_out, st, run_flag);
    if (gaps_done) *gaps_done = gap_out != nullptr;
    if (rc) return rc;
    AFFMAE_LAUNCH_CHECK("seg_sort_cl_kernel");
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


}  // namespace affmae_b200
