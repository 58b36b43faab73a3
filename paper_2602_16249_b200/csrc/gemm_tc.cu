// Hand-written tcgen05 GEMM for the training step's dense layers:
//
//   D[M, N] = A[M, K] · B[N, K]^T   (bf16 operands, fp32 accumulation in TMEM)
//
// with the epilogues the step needs fused into the TMEM read-back:
//   kStore     y   = acc (+ bias[n])                               bf16
//   kGeluAux   pre = acc + bias[n] (bf16), y = GELU(pre)            bf16, bf16
//   kAdd       y   = acc + bias[n] + c[m, n]                        bf16
//   kGeluBwd   y   = acc · GELU'(pre[m, n])                          bf16
//   kF32       y   = acc (+ beta · y)                               fp32
//   kGelu      y   = GELU(acc + bias[n])  (fp32 pre-activation)     bf16
// This is the reference Tape's matmul + bias (+ gelu_erf) (proj/src/tape.cpp:24-114) and its
// VJPs: the forward x W^T (A = x K-major, B = W [N, K] K-major), the input gradient dY W
// (B = W read N-major), the weight gradient dY^T X (A = dY^T and B = X both read M/N-major).
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: 128x64 A and BNx64 B tiles (128-byte swizzle) into a
//               kStages-deep shared-memory ring, one mbarrier (complete_tx) per stage
//   warp 1      TMEM allocator + MMA issuer: one thread issues tcgen05.mma.cta_group::1
//               (M = 128, N = BN, K = 16; cta_group::2 / M = 256 for CTA pairs) from
//               shared-memory descriptors into one of two TMEM accumulators, tcgen05.commit
//               frees the ring slot / signals the epilogue
//   epilogue    8 warps (16 for the erf-bound GELU epilogues): tcgen05.ld 32x32b.x32 (warp w
//               reads TMEM lanes 32·(w%4)..), the fused elementwise op in fp32, TMA stores of
//               32 x 128 B boxes; the accumulator is released as soon as its last columns are
//               read, so tile t's epilogue overlaps tile t+1's MMAs
//   column sums one more warp in the weight-gradient form: the bias gradient from the A tiles
// Work items are (split, m-block, n-block) with m-block outermost within a split, so the
// CTAs working at one time share A rows through L2.  The weight gradient's long K (= tokens)
// is split over `splits` work ranges (multiples of 64) written as fp32 partials.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace affmae_b200 {
namespace tc {

constexpr int BM = 128, BK = 64, UK = 16;
constexpr int kStageBuf = 32 * 128;  // one epilogue staging buffer: 32 rows x 128 B

enum Epi { kStore = 0, kGeluAux = 1, kAdd = 2, kGeluBwd = 3, kF32 = 4, kGelu = 5 };
// epilogue warps: the erf-bound GELU epilogues get four per TMEM lane quarter (they bound the
// thin-K fc1 forward), the store-bound ones two (their staging buffers go to the operand ring)
template <int EPI>
struct EpiWarps {
    static constexpr int value = (EPI == kGeluAux || EPI == kGeluBwd || EPI == kGelu) ? 16 : 8;
};

struct Params {
    int M, N, K;
    int tiles_m, tiles_n, splits, kblocks_per_split, kblocks_total;
    const float* bias;        // [N] or null
    const __nv_bfloat16* aux;  // kAdd: c [M, N]; kGeluBwd: pre [M, N]
    void* out;                // bf16 [M, N] (kGeluAux: pre) or fp32 [splits][M, N]
    __nv_bfloat16* out2;      // kGeluAux: GELU(pre)
    float beta;
    int64_t ldo;              // row stride of out / out2 / aux (elements)
    // weight-gradient GEMMs (kF32, A read M-major = dY^T): column sums of dY over this call's
    // tokens, i.e. the bias gradient: cs_accum ? cs_out[m] += sum : cs_out[split * M + m] = sum
    float* cs_out;
    int cs_accum;
};

template <int BN, int EPI, bool PAIR = false, bool CS = false>
struct Cfg {
    // one 4 KB staging buffer per epilogue warp; the rest of the 227 KB goes to the operand ring
    static constexpr int kEpiWarps = EpiWarps<EPI>::value;
    // producer, MMA, epilogue warps (+ the column-sum warp of the weight-gradient GEMMs)
    static constexpr int kThreads = 64 + 32 * kEpiWarps + (CS ? 32 : 0);
    static constexpr int kBufs = 1;
    // a CTA of a pair holds its 128 rows of A and its half of the BN rows of B
    static constexpr int kABytes = BM * BK * 2, kBBytes = (PAIR ? BN / 2 : BN) * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (227 * 1024 - kEpiWarps * kBufs * kStageBuf - 2048) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr size_t kSmem =
        size_t(kStages) * kStageBytes + size_t(kEpiWarps) * kBufs * kStageBuf + 1024 /*align*/ + 256 /*barriers*/;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// parity wait; a pipeline bug traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t done = 0, spins = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return;
        if (++spins > (1u << 26)) {
            printf("tc_gemm: mbarrier wait timed out (block %d thread %d bar %u parity %u)\n", blockIdx.x, threadIdx.x, a,
                   parity);
            __trap();
        }
    }
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptors, 128-byte swizzle (SmemDescriptor, cute/arch/mma_sm100_desc.hpp):
//   K-major:  rows of 64 K-elements (128 B), 8-row groups 1024 B apart (SBO), LBO unused
//   MN-major: rows of 64 M/N-elements (128 B) per k, 8-k groups 1024 B apart (SBO), 64-wide
//             M/N chunks BK·128 B apart (LBO)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, bool mn_major) {
    const uint64_t lbo = mn_major ? uint64_t(BK * 128 / 16) : 1ull;
    return uint64_t((addr >> 4) & 0x3FFF) | (lbo << 16) | (uint64_t(1024 / 16) << 32) | (1ull << 46) | (2ull << 61);
}
// advance to the k-th 16-element slice of a 64-wide K block
__device__ __forceinline__ uint64_t sdesc_k(uint64_t d, int k, bool mn_major) {
    return d + uint64_t(mn_major ? (k * UK * 128) >> 4 : (k * UK * 2) >> 4);
}

// erf for the GELU epilogues (they bound the fc1 forward, ncu: tensor pipe 27 %): Abramowitz &
// Stegun 7.1.26, |error| <= 1.5e-7 (+ the approximate reciprocal / exponential, ~1e-7
// relative) against libm erff's branchy polynomial -- one MUFU.RCP, one MUFU.EX2 and six FMAs;
// e = exp(-z^2) is handed back for the derivative.  The results are rounded to bf16.
__device__ __forceinline__ float erf_fast(float z, float& e) {
    const float a = fabsf(z);
    float t;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, a, 1.f)));
    e = __expf(-a * a);
    const float poly =
        t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f), 0.254829592f);
    return copysignf(fmaf(-poly, e, 1.f), z);
}
// GELU(x) = x Phi(x) (the reference's gelu_erf) and its derivative Phi(x) + x phi(x)
__device__ __forceinline__ float gelu_f(float x) {
    float e;
    return 0.5f * x * (1.f + erf_fast(x * 0.70710678118654752f, e));
}
__device__ __forceinline__ float gelu_grad(float x) {
    float e;  // exp(-x^2 / 2)
    const float cdf = 0.5f * (1.f + erf_fast(x * 0.70710678118654752f, e));
    return fmaf(x * 0.39894228040143268f, e, cdf);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------------- kernel
struct Maps {
    CUtensorMap a, b;
    CUtensorMap out;   // bf16 box {64, 32} / fp32 box {32, 32}, 128-byte swizzle, [splits][M][ldo]
    CUtensorMap out2;  // kGeluAux: GELU(pre)
    CUtensorMap aux;   // kAdd / kGeluBwd: bf16 box {64, 32}
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// CTA-pair TMA load: the data lands in this CTA's shared memory, the transaction bytes are
// counted on `bar`, a shared::cluster address that may be the leader CTA's barrier
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// shared::cluster address of this CTA's variable `a` in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t a) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on the barrier at the same offset in both CTAs of the pair once the pair's MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"(uint16_t(3))
        : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// 16-byte chunk c of row r in a 32 x 128 B staging buffer written / read by TMA with the
// 128-byte swizzle (Swizzle<3,4,3> on a 1024-byte aligned base)
__device__ __forceinline__ uint32_t swz(int r, int c) { return uint32_t(r * 128 + ((c ^ (r & 7)) << 4)); }

// PAIR: a thread-block cluster of 2 CTAs on one TPC computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (UMMA M = 256): CTA r holds rows 128 r.. of A and half of the BN
// rows of B, the leader (rank 0) issues the MMAs for both SMs, each SM's TMEM receives its 128
// rows of D.  Per SM that halves the shared-memory and L2 traffic of B.  Protocol: the leader's
// full barrier counts the bytes of both CTAs (their TMA loads signal it), the leader's commits
// arrive on both CTAs' empty / tfull barriers, both CTAs' epilogue warps arrive on the leader's
// tempty barrier.
template <int BN, int EPI, bool A_MN, bool B_MN, bool PAIR>
__global__ void __launch_bounds__(Cfg<BN, EPI, PAIR, EPI == kF32 && A_MN && !PAIR>::kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ Maps maps, Params p) {
    constexpr bool MC = PAIR;
    // CS: the weight gradient's A tile (dY^T, M-major) also feeds a column-sum warp -- the bias
    // gradient comes out of the operand ring instead of a second pass over dY
    constexpr bool CS = EPI == kF32 && A_MN && !PAIR;
    using C = Cfg<BN, EPI, PAIR, CS>;
    constexpr int kEpiWarps = C::kEpiWarps;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_smem = smem + size_t(C::kStages) * C::kStageBytes;  // kEpiWarps x kBufs x 4 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(stage_smem + kEpiWarps * C::kBufs * kStageBuf);
    // full[S], empty[S], tfull[2], tempty[2], aux[8], then the TMEM base address slot
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4 + kEpiWarps);
    const uint32_t smem_base = smem_u32(smem);
    const uint32_t bar_base = smem_u32(bars);
    auto full = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto empty = [&](int s) { return bar_base + 8u * uint32_t(C::kStages + s); };
    auto tfull = [&](int s) { return bar_base + 8u * uint32_t(2 * C::kStages + s); };
    auto tempty = [&](int s) { return bar_base + 8u * uint32_t(2 * C::kStages + 2 + s); };
    auto auxbar = [&](int e) { return bar_base + 8u * uint32_t(2 * C::kStages + 4 + e); };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(full(s), 1);
            mbar_init(empty(s), CS ? 2 : 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(tfull(s), 1);
            mbar_init(tempty(s), PAIR ? 2 * kEpiWarps : kEpiWarps);
        }
        for (int e = 0; e < kEpiWarps; ++e) mbar_init(auxbar(e), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.out)) : "memory");
    }
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(uint32_t(C::kTmemCols))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(uint32_t(C::kTmemCols))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    fence_before();
    if (MC)
        cluster_sync();  // the peer's barriers are initialised before any multicast reaches them
    else
        __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // work items (split, m-group, n-block); an m-group is one m-block, or a pair with MC
    const int rank = MC ? int(blockIdx.x & 1) : 0;
    const int cid = MC ? int(blockIdx.x >> 1) : int(blockIdx.x);
    const int ncl = MC ? int(gridDim.x >> 1) : int(gridDim.x);
    const int mgroups = MC ? (p.tiles_m + 1) / 2 : p.tiles_m;
    const int tiles = mgroups * p.tiles_n;
    const int work = tiles * p.splits;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int w = cid; w < work; w += ncl) {
                const int split = w / tiles, t = w - split * tiles;
                const int mg = t / p.tiles_n, nb = t - mg * p.tiles_n;
                const int mb = MC ? 2 * mg + rank : mg;
                const int kb0 = split * p.kblocks_per_split;
                const int kb1 = min(kb0 + p.kblocks_per_split, p.kblocks_total);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty(stage), phase ^ 1);
                    const uint32_t sa = smem_base + uint32_t(stage) * C::kStageBytes;
                    const uint32_t sb = sa + C::kABytes;
                    if (PAIR) {
                        // both CTAs' loads count on the leader's full barrier
                        const uint32_t fb = mapa(full(stage), 0);
                        if (rank == 0) mbar_expect_tx(full(stage), 2 * C::kStageBytes);
                        if (A_MN) {
#pragma unroll
                            for (int c = 0; c < BM / 64; ++c)
                                tma_load_3d_pair(sa + c * (BK * 128), &maps.a, mb * BM + 64 * c, kb * BK, 0, fb);
                        } else {
                            tma_load_3d_pair(sa, &maps.a, kb * BK, mb * BM, 0, fb);
                        }
                        if (B_MN) {
#pragma unroll
                            for (int c = 0; c < BN / 128; ++c)
                                tma_load_3d_pair(sb + c * (BK * 128), &maps.b, nb * BN + rank * (BN / 2) + 64 * c,
                                                 kb * BK, 0, fb);
                        } else {
                            tma_load_3d_pair(sb, &maps.b, kb * BK, nb * BN + rank * (BN / 2), 0, fb);
                        }
                        if (++stage == C::kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    mbar_expect_tx(full(stage), C::kStageBytes);
                    if (A_MN) {
#pragma unroll
                        for (int c = 0; c < BM / 64; ++c)
                            tma_load_3d(sa + c * (BK * 128), &maps.a, mb * BM + 64 * c, kb * BK, 0, full(stage));
                    } else {
                        tma_load_3d(sa, &maps.a, kb * BK, mb * BM, 0, full(stage));
                    }
                    if (B_MN) {
#pragma unroll
                        for (int c = 0; c < BN / 64; ++c)
                            tma_load_3d(sb + c * (BK * 128), &maps.b, nb * BN + 64 * c, kb * BK, 0, full(stage));
                    } else {
                        tma_load_3d(sb, &maps.b, kb * BK, nb * BN, 0, full(stage));
                    }
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (CS && warp == 2 + kEpiWarps) {
        // column sums of the A tile (k rows x 128 m, two 64-wide M-major chunks, 128-byte
        // swizzle): lane l owns m = 4l .. 4l+3 and reads them as one 8-byte load per k row; every
        // ring slot is released by this warp as well as by the MMA commit
        int stage = 0;
        uint32_t phase = 0;
        const int c = lane >> 4, j = (lane & 15) >> 1;
        for (int w = cid; w < work; w += ncl) {
            const int split = w / tiles, t = w - split * tiles;
            const int mg = t / p.tiles_n, nb = t - mg * p.tiles_n;
            const int mb = MC ? 2 * mg + rank : mg;
            const int kb0 = split * p.kblocks_per_split;
            const int kb1 = min(kb0 + p.kblocks_per_split, p.kblocks_total);
            const bool active = p.cs_out && nb == 0;
            float a4[4] = {0.f, 0.f, 0.f, 0.f};
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(full(stage), phase);
                if (active) {
                    const uint8_t* tile = smem + size_t(stage) * C::kStageBytes + c * (BK * 128) + 8 * (lane & 1);
#pragma unroll 8
                    for (int r = 0; r < BK; ++r) {
                        const uint2 v = *reinterpret_cast<const uint2*>(tile + r * 128 + ((j ^ (r & 7)) << 4));
                        const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
                        const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
                        a4[0] += f0.x;
                        a4[1] += f0.y;
                        a4[2] += f1.x;
                        a4[3] += f1.y;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty(stage));
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (active) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = mb * BM + 4 * lane + i;
                    if (m < p.M) {
                        if (p.cs_accum)
                            p.cs_out[m] += a4[i];
                        else
                            p.cs_out[int64_t(split) * p.M + m] = a4[i];
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // instruction descriptor (InstrDescriptor): fp32 D, bf16 A / B, majors, N >> 3, M >> 4
            constexpr uint32_t kUmmaM = PAIR ? 2 * BM : BM;
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(A_MN) << 15) |
                                   (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) | ((kUmmaM >> 4) << 24);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int w = cid; w < work; w += ncl) {
                const int split = w / tiles;
                const int kb0 = split * p.kblocks_per_split;
                const int kb1 = min(kb0 + p.kblocks_per_split, p.kblocks_total);
                mbar_wait(tempty(acc), acc_phase ^ 1);
                fence_after();
                const uint32_t tmem_d = tmem_base + uint32_t(acc * BN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(full(stage), phase);
                    fence_after();
                    const uint32_t sa = smem_base + uint32_t(stage) * C::kStageBytes;
                    const uint64_t da = sdesc(sa, A_MN), db = sdesc(sa + C::kABytes, B_MN);
#pragma unroll
                    for (int k = 0; k < BK / UK; ++k) {
                        if (PAIR)
                            mma_bf16_pair(tmem_d, sdesc_k(da, k, A_MN), sdesc_k(db, k, B_MN), idesc,
                                          (kb > kb0 || k > 0) ? 1u : 0u);
                        else
                            mma_bf16(tmem_d, sdesc_k(da, k, A_MN), sdesc_k(db, k, B_MN), idesc,
                                     (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    if (PAIR)
                        mma_commit_pair(empty(stage));
                    else
                        mma_commit(empty(stage));
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (PAIR)
                    mma_commit_pair(tfull(acc));
                else
                    mma_commit(tfull(acc));
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // Epilogue: a warp owns 32 accumulator rows (its TMEM lane quarter) and, per unit, 128
        // bytes of output columns (64 bf16 / 32 fp32); it converts its rows into a swizzled
        // 32 x 128 B staging buffer and one lane hands the buffer to a TMA store, so the global
        // writes are whole lines (the M / N tails are clipped by the tensor map).
        constexpr bool kF32Out = EPI == kF32;
        constexpr int kCols = kF32Out ? 32 : 64;  // columns per unit (one 128-byte TMA box)
        constexpr int kUnits = BN / kCols;
        constexpr int kSlots = kEpiWarps / 4;     // warps per lane quarter
        constexpr bool kAux = EPI == kAdd || EPI == kGeluBwd;
        const int ew = warp - 2;       // 0 .. kEpiWarps-1
        const int quarter = warp & 3;  // TMEM lanes 32·quarter .. +31 (tcgen05.ld lane rule)
        const int slot = ew >> 2;      // units slot, slot + kSlots, ...
        const uint32_t buf0 = smem_u32(stage_smem) + uint32_t(ew) * C::kBufs * kStageBuf;
        uint8_t* gbuf0 = stage_smem + size_t(ew) * C::kBufs * kStageBuf;
        uint4 pre[EPI == kGeluAux ? 8 : 1];  // kGeluAux: the unit's bf16 pre-activations
        auto release = [&](int a) {
            fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR)
                    mbar_arrive_cluster(mapa(tempty(a), 0));
                else
                    mbar_arrive(tempty(a));
            }
        };
        int acc = 0;
        uint32_t acc_phase = 0, aux_phase = 0;
        for (int w = cid; w < work; w += ncl) {
            const int split = w / tiles, t = w - split * tiles;
            const int mg = t / p.tiles_n, nb = t - mg * p.tiles_n;
            const int mb = MC ? 2 * mg + rank : mg;
            const int row0 = mb * BM + 32 * quarter;
            mbar_wait(tfull(acc), acc_phase);
            fence_after();
            if (slot >= kUnits) release(acc);
#pragma unroll 1
            for (int u = slot; u < kUnits; u += kSlots) {
                const int n0 = nb * BN + kCols * u;
                const bool last = u + kSlots >= kUnits;  // this warp's last unit of the tile
                // the staging buffers are free once the previous unit's TMA stores have read them
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
                if (kAux && n0 < p.N && lane == 0) {
                    mbar_expect_tx(auxbar(ew), kStageBuf);
                    tma_load_3d(buf0, &maps.aux, n0, row0, 0, auxbar(ew));
                }
                if (n0 >= p.N) {  // warp-uniform: nothing to store, only the accumulator to release
                    if (last) release(acc);
                    continue;
                }
                if (kAux) {
                    mbar_wait(auxbar(ew), aux_phase);
                    aux_phase ^= 1;
                }
                // 32 columns at a time: a lane holds one row's 32 fp32 values, so four epilogue
                // warps per lane quarter fit the register file
#pragma unroll
                for (int hh = 0; hh < kCols / 32; ++hh) {
                    float v[32];
                    tmem_ld32(tmem_base + (uint32_t(32 * quarter) << 16) + uint32_t(acc * BN + kCols * u + 32 * hh), v);
                    if (last && hh + 1 == kCols / 32) release(acc);
                    const int c0 = n0 + 32 * hh;
                    if (p.bias && EPI != kGeluBwd && EPI != kF32) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            if (c0 + j < p.N) {
                                const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + c0 + j));
                                v[j] += b.x;
                                v[j + 1] += b.y;
                                v[j + 2] += b.z;
                                v[j + 3] += b.w;
                            }
                        }
                    }
                    if (kF32Out) {
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            *reinterpret_cast<float4*>(gbuf0 + swz(lane, c)) =
                                make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                        continue;
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const int c = 4 * hh + cc;  // 16-byte chunk of the 128-byte row
                        float* x = v + 8 * cc;
                        if (kAux) {
                            // the row's own aux chunk (same lane, read before it is overwritten)
                            const uint4 a = *reinterpret_cast<const uint4*>(gbuf0 + swz(lane, c));
                            const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 f = __bfloat1622float2(ah[e]);
                                if (EPI == kAdd) {
                                    x[2 * e] += f.x;
                                    x[2 * e + 1] += f.y;
                                } else {
                                    x[2 * e] *= gelu_grad(f.x);
                                    x[2 * e + 1] *= gelu_grad(f.y);
                                }
                            }
                        }
                        if (EPI == kGelu) {
#pragma unroll
                            for (int e = 0; e < 8; ++e) x[e] = gelu_f(x[e]);
                        }
                        uint4 r;
                        r.x = pack_bf16(x[0], x[1]);
                        r.y = pack_bf16(x[2], x[3]);
                        r.z = pack_bf16(x[4], x[5]);
                        r.w = pack_bf16(x[6], x[7]);
                        *reinterpret_cast<uint4*>(gbuf0 + swz(lane, c)) = r;
                        if (EPI == kGeluAux) pre[c & (EPI == kGeluAux ? 7 : 0)] = r;
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    if (kF32Out && p.beta != 0.f)
                        tma_reduce_add_3d(&maps.out, buf0, n0, row0, split);
                    else
                        tma_store_3d(&maps.out, buf0, n0, row0, split);
                    bulk_commit();
                }
                if (EPI == kGeluAux) {
                    // GELU of the stored (bf16-rounded) pre-activation, as the backward sees it,
                    // through the same staging buffer once the pre-activation store has read it
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&pre[c & 7]);
                        uint4 y;
                        uint32_t* yw = reinterpret_cast<uint32_t*>(&y);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 f = __bfloat1622float2(rh[e]);
                            yw[e] = pack_bf16(gelu_f(f.x), gelu_f(f.y));
                        }
                        *reinterpret_cast<uint4*>(gbuf0 + swz(lane, c)) = y;
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&maps.out2, buf0, n0, row0, 0);
                        bulk_commit();
                    }
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) bulk_wait0();
    }
    __syncwarp();
    fence_before();
    if (MC)
        cluster_sync();  // no CTA leaves while its peer may still multicast into it
    else
        __syncthreads();
    if (warp == 1) {
        __syncwarp();
        fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(uint32_t(C::kTmemCols))
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(uint32_t(C::kTmemCols))
                         : "memory");
    }
}

// --------------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// row-major [layers][rows][cols] (row stride ld elements, layer stride rows·ld), 128-byte
// swizzle, box = 128 bytes of columns x box_rows rows x 1 layer
int make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows, bool f32 = false,
             int64_t layers = 1) {
    auto enc = encoder();
    if (!enc) return fail(AFFMAE_ECUDA, "gemm: cuTensorMapEncodeTiled unavailable");
    const int64_t es = f32 ? 4 : 2;
    if (reinterpret_cast<uintptr_t>(ptr) % 16 || (ld * es) % 16)
        return fail(AFFMAE_EUNSUPPORTED, "gemm: operands need 16-byte aligned rows");
    cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(rows), cuuint64_t(layers)};
    cuuint64_t strides[2] = {cuuint64_t(ld * es), cuuint64_t(rows * ld * es)};
    cuuint32_t box[3] = {cuuint32_t(128 / es), cuuint32_t(box_rows), 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                           const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(AFFMAE_ECUDA, "gemm: cuTensorMapEncodeTiled failed");
    return AFFMAE_OK;
}

template <int BN, int EPI, bool A_MN, bool B_MN, bool MC>
int launch(const Maps& maps, const Params& p, cudaStream_t st) {
    using C = Cfg<BN, EPI, MC, EPI == kF32 && A_MN && !MC>;
    auto kern = tc_gemm_kernel<BN, EPI, A_MN, B_MN, MC>;
    // the shared-memory opt-in is per device: set it once for every device this process uses
    static std::mutex mu;
    static uint64_t done_mask = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_status(cudaGetLastError(), "gemm: device");
    {
        std::lock_guard<std::mutex> lock(mu);
        const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
        if (!bit || !(done_mask & bit)) {
            const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
            if (e != cudaSuccess) return cuda_status(e, "gemm: smem attribute");
            done_mask |= bit;
        }
    }
    const int groups = MC ? (p.tiles_m + 1) / 2 : p.tiles_m;
    const int work = groups * p.tiles_n * p.splits;
    const int sms = device_sms();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(MC ? 2 * std::min(work, sms / 2) : std::min(work, sms)));
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = MC ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, maps, p);
    if (e != cudaSuccess) return cuda_status(e, "tc_gemm_kernel launch");
    return AFFMAE_OK;
}

template <int EPI, bool A_MN, bool B_MN>
int dispatch_bn(int bn, bool mc, const Maps& maps, const Params& p, cudaStream_t st) {
    if (bn == 256)
        return mc ? launch<256, EPI, A_MN, B_MN, true>(maps, p, st) : launch<256, EPI, A_MN, B_MN, false>(maps, p, st);
    if (bn == 128)
        return mc ? launch<128, EPI, A_MN, B_MN, true>(maps, p, st) : launch<128, EPI, A_MN, B_MN, false>(maps, p, st);
    return launch<64, EPI, A_MN, B_MN, false>(maps, p, st);
}

int pick_bn(int64_t n) {
    if (n <= 64) return 64;
    if (n <= 128) return 128;
    // least padding; ties to the wider tile
    const int64_t p256 = (n + 255) / 256 * 256, p128 = (n + 127) / 128 * 128;
    return p256 <= p128 ? 256 : 128;
}

}  // namespace tc

// D[M, N] = op(A) op(B)^T (see the file header).
//   a_mn = 0: A is x [M, K] row-major (lda = K);  a_mn = 1: A is read from a [K, M] row-major buffer
//   b_mn = 0: B is W [N, K] row-major;            b_mn = 1: B is read from a [K, N] row-major buffer
// splits > 1 (kF32 only): K is cut into `splits` ranges, split s writes out + s·M·ldo.
int tc_gemm(const void* a, bool a_mn, const void* b, bool b_mn, int64_t M, int64_t N, int64_t K, int epi,
            const float* bias, const void* aux, void* out, void* out2, float beta, int64_t ldo, int splits,
            cudaStream_t st, float* cs_out, int cs_accum) {
    using namespace tc;
    if (!a || !b || !out) return fail(AFFMAE_ECONFIG, "gemm: null pointer");
    if (M < 1 || N < 1 || K < 1 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
        return fail(AFFMAE_ECONFIG, "gemm: bad shape");
    // 16-byte aligned rows for every TMA view: N (output / N-major B rows), K of a K-major
    // operand, M of an M-major A
    if (N % 8 || ((!a_mn || !b_mn) && K % 8) || (a_mn && M % 8))
        return fail(AFFMAE_EUNSUPPORTED, "gemm: N, K of a K-major operand and M of an M-major A must be multiples of 8");
    if ((epi == kGeluAux && !out2) || ((epi == kAdd || epi == kGeluBwd) && !aux))
        return fail(AFFMAE_ECONFIG, "gemm: epilogue operand missing");
    if (splits < 1 || (splits > 1 && epi != kF32)) return fail(AFFMAE_ECONFIG, "gemm: split-K needs the fp32 epilogue");
    if (ldo < N || ldo % 8) return fail(AFFMAE_ECONFIG, "gemm: bad output stride");
    if (bias && reinterpret_cast<uintptr_t>(bias) % 16)
        return fail(AFFMAE_EUNSUPPORTED, "gemm: the bias must be 16-byte aligned (the epilogue reads it as float4)");
    const int bn = pick_bn(N);
    Maps maps;
    int rc;
    if ((rc = a_mn ? make_map(&maps.a, a, K, M, M, BK) : make_map(&maps.a, a, M, K, K, BM))) return rc;
    // CTA pairs (UMMA M = 256 over two SMs) when there are two m-blocks to pair and B splits
    // into two halves
    // into two halves.  Measured (profiles/r02k_gemm_ab.txt): pairs win once the main loop
    // dominates -- K >= 512 with 256-wide tiles -- and lose on thin K, on the GELU epilogues
    // (epilogue-bound) and on the split-K weight gradient
    const bool mc = !a_mn && bn == 256 && K >= 512 && (M + BM - 1) / BM >= 2 &&
                    (epi == kStore || epi == kAdd || epi == kF32);
    if ((rc = b_mn ? make_map(&maps.b, b, K, N, N, BK) : make_map(&maps.b, b, N, K, K, mc ? bn / 2 : bn))) return rc;
    Params p{};
    p.M = int(M);
    p.N = int(N);
    p.K = int(K);
    p.tiles_m = int((M + BM - 1) / BM);
    p.tiles_n = int((N + bn - 1) / bn);
    p.kblocks_total = int((K + BK - 1) / BK);
    p.splits = std::min(splits, p.kblocks_total);
    p.kblocks_per_split = (p.kblocks_total + p.splits - 1) / p.splits;
    p.splits = (p.kblocks_total + p.kblocks_per_split - 1) / p.kblocks_per_split;
    p.bias = bias;
    p.aux = static_cast<const __nv_bfloat16*>(aux);
    p.out = out;
    p.out2 = static_cast<__nv_bfloat16*>(out2);
    p.beta = beta;
    p.ldo = ldo;
    if (cs_out && !(epi == kF32 && a_mn)) return fail(AFFMAE_ECONFIG, "gemm: column sums need the weight-gradient form");
    p.cs_out = cs_out;
    p.cs_accum = cs_accum;
    if (splits > 1 && p.splits != splits) return fail(AFFMAE_ECONFIG, "gemm: split count does not divide K blocks");
    if (epi == kF32 && beta != 0.f && beta != 1.f) return fail(AFFMAE_EUNSUPPORTED, "gemm: fp32 beta must be 0 or 1");
    if ((rc = make_map(&maps.out, out, M, N, ldo, 32, epi == kF32, p.splits))) return rc;
    maps.out2 = maps.out;
    maps.aux = maps.out;
    if (epi == kGeluAux && (rc = make_map(&maps.out2, out2, M, N, ldo, 32))) return rc;
    if ((epi == kAdd || epi == kGeluBwd) && (rc = make_map(&maps.aux, aux, M, N, ldo, 32))) return rc;
    const int key = (a_mn ? 2 : 0) | (b_mn ? 1 : 0);
    switch (epi) {
        case kStore:
            if (key == 0) return dispatch_bn<kStore, false, false>(bn, mc, maps, p, st);
            if (key == 1) return dispatch_bn<kStore, false, true>(bn, mc, maps, p, st);
            break;
        case kGeluAux:
            if (key == 0) return dispatch_bn<kGeluAux, false, false>(bn, mc, maps, p, st);
            break;
        case kGelu:
            if (key == 0) return dispatch_bn<kGelu, false, false>(bn, mc, maps, p, st);
            break;
        case kAdd:
            if (key == 0) return dispatch_bn<kAdd, false, false>(bn, mc, maps, p, st);
            break;
        case kGeluBwd:
            if (key == 1) return dispatch_bn<kGeluBwd, false, true>(bn, mc, maps, p, st);
            break;
        case kF32:
            if (key == 1) return dispatch_bn<kF32, false, true>(bn, mc, maps, p, st);
            if (key == 3) return dispatch_bn<kF32, true, true>(bn, mc, maps, p, st);
            break;
        default:
            break;
    }
    return fail(AFFMAE_EUNSUPPORTED, "gemm: epilogue / operand-major combination not instantiated");
}

// split count that fills the GPU: splits of >= 512 tokens each
int tc_gemm_pick_splits(int64_t M, int64_t N, int64_t K) {
    const int64_t tiles = ((M + tc::BM - 1) / tc::BM) * ((N + tc::pick_bn(N) - 1) / tc::pick_bn(N));
    const int64_t kb = (K + tc::BK - 1) / tc::BK;
    int64_t s = std::max<int64_t>(1, device_sms() / std::max<int64_t>(tiles, 1));
    s = std::min<int64_t>(s, std::max<int64_t>(1, kb / 8));
    // make the split an exact partition of the K blocks (tc_gemm requires it)
    while (s > 1) {
        const int64_t per = (kb + s - 1) / s;
        if ((kb + per - 1) / per == s) break;
        --s;
    }
    return int(s);
}

}  // namespace affmae_b200
