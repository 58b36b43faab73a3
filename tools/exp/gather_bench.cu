// Gather microbenchmark: 64-byte head slices of random token rows into shared
// memory, three ways -- per-lane 16-B cp.async (LDGSTS, swizzled), per-row
// cp.async.bulk (TMA unit, padded 80-B stride), and TMA tile::gather4 (4 rows
// per op, 64B hardware swizzle).  One warp per CTA, persistent, items of 48
// rows, two-stage pipeline; a checksum of the landed tiles checks all three.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int ROWS = 48, HD = 32, HEADS = 4, LD = HEADS * HD;  // bf16 elements per token row

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ uint32_t consume(const uint8_t* t, int stride, int lane) {
    // every lane reads 16 B of each of the 48 rows (3 rows per lane-group)
    uint32_t x = 0;
    for (int r = lane >> 2; r < ROWS; r += 8) {
        uint4 v = *reinterpret_cast<const uint4*>(t + r * stride + (lane & 3) * 16);
        x ^= v.x + 3 * v.y + 5 * v.z + 7 * v.w + r;
    }
    return x;
}
// swizzled (64B pattern) read of logical chunk c of row r
__device__ __forceinline__ int swz(int r, int c) { return r * 64 + ((c ^ ((r >> 1) & 3)) << 4); }
__device__ __forceinline__ uint32_t consume_swz(const uint8_t* t, int lane) {
    uint32_t x = 0;
    for (int r = lane >> 2; r < ROWS; r += 8) {
        uint4 v = *reinterpret_cast<const uint4*>(t + swz(r, lane & 3));
        x ^= v.x + 3 * v.y + 5 * v.z + 7 * v.w + r;
    }
    return x;
}

__global__ void k_ldgsts(const __nv_bfloat16* src, const int* idx, int items, uint32_t* out) {
    __shared__ __align__(1024) uint8_t tile[2][ROWS * 64];
    const int lane = threadIdx.x, h = blockIdx.y;
    uint32_t acc = 0;
    auto issue = [&](int it, int buf) {
        const int sub = lane >> 2, ch = lane & 3;
        for (int j = 0; j < ROWS / 8; ++j) {
            const int r = sub + 8 * j;
            const int t = idx[it * ROWS + r];
            const char* g = reinterpret_cast<const char*>(src + size_t(t) * LD + h * HD) + ch * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(tile[buf] + swz(r, ch))), "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int it = blockIdx.x, buf = 0;
    if (it < items) issue(it, 0);
    for (; it < items; it += gridDim.x) {
        const int nx = it + gridDim.x;
        if (nx < items) issue(nx, buf ^ 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        acc += consume_swz(tile[buf], lane);
        __syncwarp();
        buf ^= 1;
    }
    atomicAdd(out, acc);
}

__global__ void k_bulk(const __nv_bfloat16* src, const int* idx, int items, uint32_t* out) {
    __shared__ __align__(1024) uint8_t tile[2][ROWS * 80];
    __shared__ uint64_t bar[2];
    const int lane = threadIdx.x, h = blockIdx.y;
    if (lane == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0, ph[2] = {0, 0};
    auto issue = [&](int it, int buf) {
        if (lane == 0) mbar_expect(&bar[buf], ROWS * 64);
        __syncwarp();
        for (int r = lane; r < ROWS; r += 32) {
            const int t = idx[it * ROWS + r];
            const void* g = src + size_t(t) * LD + h * HD;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];" ::"r"(su32(tile[buf] + r * 80)), "l"(g), "r"(su32(&bar[buf])) : "memory");
        }
    };
    int it = blockIdx.x, buf = 0;
    if (it < items) issue(it, 0);
    for (; it < items; it += gridDim.x) {
        const int nx = it + gridDim.x;
        if (nx < items) issue(nx, buf ^ 1);
        mbar_wait(&bar[buf], ph[buf]);
        ph[buf] ^= 1;
        acc += consume(tile[buf], 80, lane);
        __syncwarp();
        buf ^= 1;
    }
    atomicAdd(out, acc);
}

__global__ void k_gather4(const __grid_constant__ CUtensorMap tm, const int* idx, int items, uint32_t* out) {
    __shared__ __align__(1024) uint8_t tile[2][ROWS * 64];
    __shared__ uint64_t bar[2];
    const int lane = threadIdx.x, h = blockIdx.y;
    if (lane == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0, ph[2] = {0, 0};
    auto issue = [&](int it, int buf) {
        if (lane == 0) mbar_expect(&bar[buf], ROWS * 64);
        __syncwarp();
        if (lane < ROWS / 4) {
            const int4 t = *reinterpret_cast<const int4*>(idx + it * ROWS + 4 * lane);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(tile[buf] + lane * 256)),
                "l"(&tm), "r"(h * HD), "r"(t.x), "r"(t.y), "r"(t.z), "r"(t.w), "r"(su32(&bar[buf]))
                : "memory");
        }
    };
    int it = blockIdx.x, buf = 0;
    if (it < items) issue(it, 0);
    for (; it < items; it += gridDim.x) {
        const int nx = it + gridDim.x;
        if (nx < items) issue(nx, buf ^ 1);
        mbar_wait(&bar[buf], ph[buf]);
        ph[buf] ^= 1;
        acc += consume_swz(tile[buf], lane);
        __syncwarp();
        buf ^= 1;
    }
    atomicAdd(out, acc);
}

int main(int argc, char** argv) {
    const int N = 524288, items = argc > 1 ? atoi(argv[1]) : 32768;
    const int window = argc > 2 ? atoi(argv[2]) : 1024;  // rows of an item drawn near item*16
    std::vector<int> hidx(size_t(items) * ROWS);
    srand(1);
    for (int i = 0; i < items; ++i)
        for (int r = 0; r < ROWS; ++r) {
            long c = long(i) * 16 + (rand() % window) - window / 2;
            hidx[size_t(i) * ROWS + r] = int(((c % N) + N) % N);
        }
    std::vector<uint16_t> hsrc(size_t(N) * LD);
    for (size_t i = 0; i < hsrc.size(); ++i) hsrc[i] = uint16_t(rand());
    __nv_bfloat16* src; int* idx; uint32_t* out;
    CK(cudaMalloc(&src, hsrc.size() * 2));
    CK(cudaMalloc(&idx, hidx.size() * 4));
    CK(cudaMalloc(&out, 16));
    CK(cudaMemcpy(src, hsrc.data(), hsrc.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(LD), cuuint64_t(N)};
    cuuint64_t strides[1] = {cuuint64_t(LD) * 2};
    cuuint32_t box[2] = {HD, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", int(cr)); return 1; }

    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[3] = {"ldgsts16", "bulk_row", "gather4"};
    for (int kind = 0; kind < 3; ++kind) {
        for (int occ : {8, 16, 24}) {
            dim3 grid(sms * occ / HEADS, HEADS);
            uint32_t sum = 0;
            float best = 1e9;
            for (int rep = 0; rep < 6; ++rep) {
                CK(cudaMemset(out, 0, 4));
                cudaEventRecord(e0);
                if (kind == 0) k_ldgsts<<<grid, 32>>>(src, idx, items, out);
                else if (kind == 1) k_bulk<<<grid, 32>>>(src, idx, items, out);
                else k_gather4<<<grid, 32>>>(tm, idx, items, out);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep) best = ms < best ? ms : best;
                CK(cudaMemcpy(&sum, out, 4, cudaMemcpyDeviceToHost));
            }
            CK(cudaGetLastError());
            const double bytes = double(items) * HEADS * ROWS * 64;
            printf("%-9s occ %2d: %8.1f us  %7.1f GB/s  %.2f Gitem-heads/s  checksum %08x\n", names[kind], occ,
                   best * 1e3, bytes / best / 1e6, items * HEADS / best / 1e6, sum);
        }
    }
    return 0;
}
