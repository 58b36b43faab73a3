// The merge's standalone functions: importance_scores
// (proj/src/merging.cpp:31-48) and merge_tokens with its layer_norm_rows
// (proj/src/merging.cpp:222-273).  The model path computes the same scorer with a
// tensor-core GEMM inside the training step (model.cu); these are the reference's free
// functions behind the C ABI.
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "model_kernels.h"

namespace affmae_b200 {
namespace {

constexpr int kScoreMaxHidden = 32;

// One thread per token in binary64 with the reference's operation order: pre_j = b1_j +
// sum_c f_c w1[c][j] (sequential in c, no contraction), GELU(erf), pre2 = b2 + sum_j g_j w2_j,
// sigmoid; rounded once to fp32 (the b32 tensor the reference writes).  The token's features
// are read once (the H accumulators advance together; each keeps its own c order).
template <int H>
__global__ void importance_scores_kernel(const float* __restrict__ feats, int64_t rows, int64_t dim,
                                         const float* __restrict__ w1, const float* __restrict__ b1,
                                         const float* __restrict__ w2, const float* __restrict__ b2, int hidden,
                                         float* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc[H];
#pragma unroll
    for (int j = 0; j < H; ++j) acc[j] = j < hidden ? double(__ldg(b1 + j)) : 0.0;
    const float* f = feats + i * dim;
    for (int64_t c = 0; c < dim; ++c) {
        const double x = double(__ldg(f + c));
        const float* wr = w1 + c * hidden;
#pragma unroll
        for (int j = 0; j < H; ++j)
            if (j < hidden) acc[j] = __dadd_rn(acc[j], __dmul_rn(x, double(__ldg(wr + j))));
    }
    double pre2 = double(__ldg(b2));
#pragma unroll
    for (int j = 0; j < H; ++j) {
        if (j >= hidden) break;
        const double g = __dmul_rn(__dmul_rn(0.5, acc[j]), __dadd_rn(1.0, erf(__dmul_rn(acc[j], 0.70710678118654752440))));
        pre2 = __dadd_rn(pre2, __dmul_rn(g, double(__ldg(w2 + j))));
    }
    out[i] = float(__ddiv_rn(1.0, __dadd_rn(1.0, exp(-pre2))));
}

__global__ void gather_retained_coords_kernel(const float2* __restrict__ coords, const int32_t* __restrict__ retained,
                                              int64_t batch, int64_t n, int64_t r, float2* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * r) return;
    const int64_t b = i / r;
    out[i] = coords[b * n + retained[i]];
}

__global__ void zero_f32_kernel(float* __restrict__ x, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = 0.f;
}

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct TokWs {
    affmae_merge_plan plan;
    uint8_t* plan_ws;
    size_t plan_ws_bytes;
    __nv_bfloat16* pooled;
    __nv_bfloat16* merged;
    float* stats;
    float* zero_bias;
    uint8_t* gemm_ws;
    size_t gemm_ws_bytes;
    size_t bytes;
};

TokWs carve_tok(int64_t batch, int64_t n, int64_t r, int64_t dim, int k_m, void* base) {
    TokWs w{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* q = p ? p + off : nullptr;
        off += al(bytes);
        return q;
    };
    w.plan.target = reinterpret_cast<int32_t*>(take(size_t(batch * n) * 4));
    w.plan.pool_idx = reinterpret_cast<int32_t*>(take(size_t(batch * r * k_m) * 4));
    w.plan.pool_dist = reinterpret_cast<double*>(take(size_t(batch * r * k_m) * 8));
    w.plan.pool_cnt = reinterpret_cast<int32_t*>(take(size_t(batch * r) * 4));
    w.plan.row_of = reinterpret_cast<int32_t*>(take(size_t(batch * n) * 4));
    w.plan_ws_bytes = merge_plan_workspace(batch, n, r);
    w.plan_ws = take(w.plan_ws_bytes);
    w.pooled = reinterpret_cast<__nv_bfloat16*>(take(size_t(batch * r * 2 * dim) * 2));
    w.merged = reinterpret_cast<__nv_bfloat16*>(take(size_t(batch * r * dim) * 2));
    w.stats = reinterpret_cast<float*>(take(size_t(batch * r) * 8));
    w.zero_bias = reinterpret_cast<float*>(take(size_t(dim) * 4));
    w.gemm_ws_bytes = linear_workspace(batch * r, dim, 2 * dim);
    w.gemm_ws = take(w.gemm_ws_bytes);
    w.bytes = off;
    return w;
}

}  // namespace

int importance_scores(const float* feats, int64_t rows, int64_t dim, const float* w1, const float* b1,
                      const float* w2, const float* b2, int hidden, float* out, void* stream) {
    if (!feats || !w1 || !b1 || !w2 || !b2 || !out) return fail(AFFMAE_ECONFIG, "importance_scores: null pointer");
    if (rows < 0 || dim < 1 || hidden < 1) return fail(AFFMAE_ECONFIG, "importance_scores: bad shape");
    if (hidden > kScoreMaxHidden) return fail(AFFMAE_EUNSUPPORTED, "importance_scores: hidden > 32 not compiled");
    if (rows == 0) return AFFMAE_OK;
    const unsigned nb = unsigned((rows + 127) / 128);
    cudaStream_t st = as_stream(stream);
    if (hidden <= 8) importance_scores_kernel<8><<<nb, 128, 0, st>>>(feats, rows, dim, w1, b1, w2, b2, hidden, out);
    else if (hidden <= 16) importance_scores_kernel<16><<<nb, 128, 0, st>>>(feats, rows, dim, w1, b1, w2, b2, hidden, out);
    else importance_scores_kernel<32><<<nb, 128, 0, st>>>(feats, rows, dim, w1, b1, w2, b2, hidden, out);
    AFFMAE_LAUNCH_CHECK("importance_scores_kernel");
    return AFFMAE_OK;
}

size_t merge_tokens_workspace(int64_t batch, int64_t n, int64_t r, int64_t dim, int k_m) {
    if (batch < 0 || n < 1 || r < 1 || dim < 1 || k_m < 1) return 0;
    return carve_tok(batch, n, r, dim, k_m, nullptr).bytes;
}

int merge_tokens(const float* coords, const void* feats, const float* scores, const int32_t* retained, int64_t batch,
                 int64_t n, int64_t r, int64_t dim, int k_m, const float* p_merge, const void* proj_wt,
                 const float* gamma, const float* beta, void* out_feats, float* out_coords, void* workspace,
                 size_t ws_bytes, void* stream) {
    if (!coords || !feats || !scores || !retained || !p_merge || !proj_wt || !gamma || !beta || !out_feats ||
        !out_coords)
        return fail(AFFMAE_ECONFIG, "merge_tokens: null pointer");
    if (batch < 0 || n < 1 || r < 1 || r > n || dim < 1 || k_m < 1)
        return fail(AFFMAE_ECONFIG, "merge_tokens: bad shape");
    if (dim % 8) return fail(AFFMAE_EUNSUPPORTED, "merge_tokens: feature width must be a multiple of 8");
    TokWs w = carve_tok(batch, n, r, dim, k_m, workspace);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "merge_tokens: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    const int64_t rows = batch * r;
    // MergePlan (bit-exact) -> pool rows [f_r ; agg] -> [2D -> D] projection -> LayerNorm rows
    if (int rc = merge_plan_build(coords, retained, batch, n, r, k_m, &w.plan, w.plan_ws, w.plan_ws_bytes, stream))
        return rc;
    if (int rc = merge_pool_fwd(reinterpret_cast<const affmae_bf16*>(feats), scores, p_merge, retained, &w.plan,
                                batch, n, r, dim, k_m, reinterpret_cast<affmae_bf16*>(w.pooled), stream))
        return rc;
    zero_f32_kernel<<<unsigned((dim + 255) / 256), 256, 0, st>>>(w.zero_bias, dim);
    AFFMAE_LAUNCH_CHECK("zero_f32_kernel");
    if (int rc = linear_fwd(w.pooled, proj_wt, w.zero_bias, rows, dim, 2 * dim, 0, w.merged, w.gemm_ws,
                            w.gemm_ws_bytes, stream))
        return rc;
    // layer_norm_rows (eps 1e-5, fp32 statistics of the bf16 projection) -- the model's row kernel
    if (int rc = mk::ln_fwd_bf(w.merged, nullptr, gamma, beta, rows, dim, static_cast<__nv_bfloat16*>(out_feats),
                               reinterpret_cast<float2*>(w.stats), st))
        return rc;
    gather_retained_coords_kernel<<<unsigned((rows + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const float2*>(coords), retained, batch, n, r, reinterpret_cast<float2*>(out_coords));
    AFFMAE_LAUNCH_CHECK("gather_retained_coords_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
