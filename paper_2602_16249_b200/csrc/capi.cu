// extern "C" entry points of libaffmae_b200.so (declared in include/affmae_b200.h)
// plus the thread-local error slot.  Argument validation mirrors the
// reference's ConfigError checks; kernels live in the other translation units.
#include <cmath>
#include <cstdio>
#include <exception>
#include <new>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace affmae_b200 {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return AFFMAE_ECUDA;
}

}  // namespace affmae_b200

using namespace affmae_b200;

// Every int-returning entry point runs under AFFMAE_GUARD: a C++ exception (a malformed
// file's std::length_error, bad_alloc, ...) becomes an error code instead of unwinding
// through the C ABI (which would std::terminate the host process).
#define AFFMAE_GUARD(...)                                                             \
    try {                                                                             \
        __VA_ARGS__                                                                   \
    } catch (const std::bad_alloc&) {                                                 \
        return fail(AFFMAE_ECONFIG, "out of host memory");                            \
    } catch (const std::exception& e) {                                               \
        return fail(AFFMAE_ECONFIG, std::string("exception: ") + e.what());          \
    } catch (...) {                                                                   \
        return fail(AFFMAE_ECONFIG, "unknown exception");                             \
    }

extern "C" {

const char* affmae_last_error(void) { return g_last_error.c_str(); }

int affmae_version(void) { return 1; }

// balanced_clusters / cluster_neighborhood closed forms (proj/src/geometry.cpp:108-156)
int affmae_cluster_geometry(affmae_cluster_geom* g) {
    if (!g) return fail(AFFMAE_ECONFIG, "cluster_geometry: null");
    if (g->batch < 0) return fail(AFFMAE_ECONFIG, "cluster_geometry: negative batch");
    if (g->tokens < 1) return fail(AFFMAE_ECONFIG, "sfc_order: empty point set");
    if (g->cluster < 1) return fail(AFFMAE_ECONFIG, "balanced_clusters: size must be >= 1");
    if (g->groups < 1) return fail(AFFMAE_ECONFIG, "cluster_neighborhood: groups must be >= 1");
    if (g->tokens > (int64_t(1) << 30)) return fail(AFFMAE_EUNSUPPORTED, "cluster_geometry: too many tokens");
    int64_t s = g->cluster < g->tokens ? g->cluster : g->tokens;
    g->n_clusters = (g->tokens + s - 1) / s;
    g->groups_eff = g->groups < g->n_clusters ? g->groups : g->n_clusters;
    g->max_size = g->tokens / g->n_clusters + (g->tokens % g->n_clusters ? 1 : 0);
    g->width = g->groups_eff * g->max_size;
    return AFFMAE_OK;
}

size_t affmae_attn_fwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    return attn_fwd_workspace(g, a);
}

int affmae_attn_fwd(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                    const affmae_attn_inputs* in, const int32_t* perm, const int32_t* nbr_cl,
                    affmae_bf16* out, float* lse, void* workspace, size_t workspace_bytes,
                    void* stream) {
    AFFMAE_GUARD(
        return attn_fwd(g, a, in, perm, nbr_cl, out, lse, workspace, workspace_bytes, stream);
    )
}

// hilbert_index (proj/src/geometry.cpp:15-30): d of cell (x, y) on a side-n grid (n a power of 2)
uint64_t affmae_hilbert_index(uint32_t n, uint32_t x, uint32_t y) { return hilbert_index_host(n, x, y); }

// flop_count_attn / flop_count_attn_dense (proj/src/attention.cpp:360-370)
uint64_t affmae_flop_count_attn(int64_t n, int64_t m, int64_t h, int64_t d) {
    if (n < 1 || m < 1 || h < 1 || d < 1) {
        fail(AFFMAE_ECONFIG, "flop_count_attn: all args must be positive");
        return 0;
    }
    const uint64_t mp = uint64_t(m) + 1;
    return 4ull * uint64_t(n) * mp * uint64_t(h) * uint64_t(d) + 6ull * uint64_t(n) * mp * uint64_t(h);
}
uint64_t affmae_flop_count_attn_dense(int64_t n, int64_t h, int64_t d) {
    if (n < 1 || h < 1 || d < 1) {
        fail(AFFMAE_ECONFIG, "flop_count_attn_dense: all args must be positive");
        return 0;
    }
    return 4ull * uint64_t(n) * uint64_t(n) * uint64_t(h) * uint64_t(d) + 6ull * uint64_t(n) * uint64_t(n) * uint64_t(h);
}

size_t affmae_attn_bwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    return attn_bwd_workspace(g, a);
}

int affmae_attn_bwd(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                    const affmae_attn_inputs* in, const affmae_cluster_index* idx,
                    const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                    affmae_attn_grads* grads, void* workspace, size_t workspace_bytes,
                    void* stream) {
    AFFMAE_GUARD(
        return attn_bwd(g, a, in, idx, out, lse, dout, grads, workspace, workspace_bytes, stream);
    )
}

size_t affmae_attn_plan_workspace(const affmae_cluster_geom* g, int with_reverse) {
    return attn_plan_workspace(g, with_reverse);
}
int affmae_attn_plan_build(const affmae_cluster_geom* g, const affmae_attn_desc* a, const float* coords,
                           const affmae_cluster_index* idx, int with_reverse, affmae_attn_plan* plan,
                           void* stream) {
    AFFMAE_GUARD(
        return attn_plan_build(g, a, coords, idx, with_reverse, plan, stream);
    )
}
size_t affmae_attn_fwd_planned_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    return attn_fwd_planned_workspace(g, a);
}
int affmae_attn_fwd_planned(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                            const affmae_attn_inputs* in, const affmae_attn_plan* plan, affmae_bf16* out,
                            float* lse, void* workspace, size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return attn_fwd_planned(g, a, in, plan, out, lse, workspace, workspace_bytes, stream);
    )
}
size_t affmae_attn_bwd_planned_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    return attn_bwd_planned_workspace(g, a);
}
int affmae_attn_bwd_planned(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                            const affmae_attn_inputs* in, const affmae_attn_plan* plan,
                            const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                            affmae_attn_grads* grads, void* workspace, size_t workspace_bytes,
                            void* stream) {
    AFFMAE_GUARD(
        return attn_bwd_planned(g, a, in, plan, out, lse, dout, grads, workspace, workspace_bytes, stream);
    )
}

size_t affmae_cluster_index_workspace(const affmae_cluster_geom* g) { return cluster_index_workspace(g); }

int affmae_cluster_index_build(const affmae_cluster_geom* g, const float* coords,
                               affmae_cluster_index* out, void* workspace, size_t workspace_bytes,
                               void* stream) {
    AFFMAE_GUARD(
        return cluster_index_build(g, coords, out, workspace, workspace_bytes, stream);
    )
}

int affmae_neighbor_expand(const affmae_cluster_geom* g, const int32_t* perm, const int32_t* nbr_cl,
                           int32_t* idx, uint8_t* valid, void* stream) {
    AFFMAE_GUARD(
        return neighbor_expand(g, perm, nbr_cl, idx, valid, stream);
    )
}

size_t affmae_sfc_order_workspace(int64_t batch, int64_t tokens) {
    return sfc_order_workspace(batch, tokens);
}

int affmae_sfc_order(const float* coords, int64_t batch, int64_t tokens, int32_t* perm,
                     void* workspace, size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return sfc_order(coords, batch, tokens, perm, workspace, workspace_bytes, stream);
    )
}

int affmae_knn(const float* queries, const float* keys, int64_t batch, int64_t n_queries,
               int64_t n_keys, int64_t k, int32_t* idx, uint8_t* valid, void* stream) {
    AFFMAE_GUARD(
        return knn(queries, keys, batch, n_queries, n_keys, k, idx, valid, stream);
    )
}

// make_interp_op forward / backward (proj/src/interpolation.cpp:192-251)
int affmae_interp_fwd(const float* queries, const float* key_coords, const affmae_bf16* feats,
                      const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t n_queries,
                      int64_t n_keys, int64_t dim, int64_t k, const float* p, double eps,
                      affmae_bf16* out, void* stream) {
    AFFMAE_GUARD(
        return interp_fwd(queries, key_coords, feats, idx, valid, batch, n_queries, n_keys, dim, k, p, eps, out,
                          stream);
    )
}
int affmae_interp_bwd(const float* queries, const float* key_coords, const affmae_bf16* feats,
                      const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t n_queries,
                      int64_t n_keys, int64_t dim, int64_t k, const float* p, double eps,
                      const affmae_bf16* dout, float* dfeats, float* dp, float* dqueries, void* stream) {
    AFFMAE_GUARD(
        return interp_bwd(queries, key_coords, feats, idx, valid, batch, n_queries, n_keys, dim, k, p, eps, dout,
                          dfeats, dp, dqueries, stream);
    )
}

size_t affmae_interp_bwd_gather_workspace(int64_t batch, int64_t n_queries, int64_t n_keys, int64_t k) {
    return interp_bwd_gather_workspace(batch, n_queries, n_keys, k);
}
int affmae_interp_bwd_gather(const float* queries, const float* key_coords, const affmae_bf16* feats,
                             const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t n_queries,
                             int64_t n_keys, int64_t dim, int64_t k, const float* p, double eps,
                             const affmae_bf16* dout, float* dfeats, float* dp, float* dqueries, void* workspace,
                             size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return interp_bwd_gather(queries, key_coords, feats, idx, valid, batch, n_queries, n_keys, dim, k, p, eps, dout,
                                 dfeats, dp, dqueries, workspace, workspace_bytes, stream);
    )
}

// device-side inputs (src/masking.cpp:34-92, src/geometry.cpp:44-50)
size_t affmae_perlin_mask_workspace(int64_t batch, int64_t h, int64_t w, int octaves, double base_freq) {
    return perlin_mask_workspace(batch, h, w, octaves, base_freq);
}
int affmae_perlin_mask(const uint64_t* seeds_host, int64_t batch, int64_t h, int64_t w, int octaves,
                       double base_freq, double persistence, double ratio, uint8_t* masked, void* workspace,
                       size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return perlin_mask(seeds_host, batch, h, w, octaves, base_freq, persistence, ratio, masked, workspace,
                           workspace_bytes, stream);
    )
}
int affmae_visible_coords(const uint8_t* masked, int64_t batch, int64_t h, int64_t w, double patch, int64_t nvis,
                          float* coords, int32_t* count, void* stream) {
    AFFMAE_GUARD(
        return visible_coords(masked, batch, h, w, patch, nvis, coords, count, stream);
    )
}

size_t affmae_synth_images_workspace(int64_t batch, int64_t size) { return synth_images_workspace(batch, size); }
int affmae_synth_images(const uint64_t* seeds_host, int64_t batch, int64_t size, double* img, void* workspace,
                        size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return synth_images(seeds_host, batch, size, img, workspace, workspace_bytes, stream);
    )
}

int affmae_patchify(const double* img, int64_t batch, int64_t h, int64_t w, int64_t patch, float* vectors,
                    void* stream) {
    AFFMAE_GUARD(
        return patchify(img, batch, h, w, patch, vectors, stream);
    )
}
int affmae_masked_rows(const uint8_t* masked, int64_t batch, int64_t cells, int64_t nmask, int32_t* rows,
                       void* stream) {
    AFFMAE_GUARD(
        return masked_rows(masked, batch, cells, nmask, rows, stream);
    )
}

// AFT1 files and checkpoints (src/tensor_io.cpp:60-105, src/pipeline.cpp:757-797)
int affmae_aft_write(const char* path, const void* dev_src, const int64_t* dims, int ndim, int dtype, void* stream) {
    AFFMAE_GUARD(
        return aft_write(path, dev_src, dims, ndim, dtype, stream);
    )
}
int affmae_aft_read_header(const char* path, int* dtype, int* ndim, int64_t* dims) {
    AFFMAE_GUARD(
        return aft_read_header(path, dtype, ndim, dims);
    )
}
int affmae_aft_read(const char* path, float* dev_dst, int64_t capacity, int64_t* numel_out, void* stream) {
    AFFMAE_GUARD(
        return aft_read(path, dev_dst, capacity, numel_out, stream);
    )
}
int affmae_checkpoint_save(const char* dir, int n, const char* const* names, const float* const* dev_vals,
                           const int64_t* const* dims, const int* ndims, const int* precs, void* stream) {
    AFFMAE_GUARD(
        return checkpoint_save(dir, n, names, dev_vals, dims, ndims, precs, stream);
    )
}
int affmae_checkpoint_load(const char* dir, int n, const char* const* names, float* const* dev_vals,
                           const int64_t* numels, void* stream) {
    AFFMAE_GUARD(
        return checkpoint_load(dir, n, names, dev_vals, numels, stream);
    )
}

// decoder attention over general neighbour rows (src/pipeline.cpp:495-535)
int affmae_gattn_fwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx,
                     const uint8_t* valid, int64_t batch, int64_t tokens, int64_t width, affmae_bf16* out,
                     float* lse, void* stream) {
    AFFMAE_GUARD(
        return gattn_fwd(a, in, idx, valid, batch, tokens, width, out, lse, stream);
    )
}
int affmae_gattn_bwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx,
                     const uint8_t* valid, int64_t batch, int64_t tokens, int64_t width, const affmae_bf16* dout,
                     affmae_bf16* dq, float* dk, float* dv, float* dblank_k, float* dblank_v, float* dw1,
                     float* db1, float* dw2, float* db2, float* dblank, void* workspace, size_t workspace_bytes,
                     void* stream) {
    AFFMAE_GUARD(
        return gattn_bwd(a, in, idx, valid, batch, tokens, width, dout, dq, dk, dv, dblank_k, dblank_v, dw1, db1, dw2,
                         db2, dblank, workspace, workspace_bytes, stream);
    )
}
size_t affmae_gattn_bwd_workspace(const affmae_attn_desc* a, int64_t batch, int64_t tokens, int64_t width) {
    return gattn_bwd_workspace(a, batch, tokens, width);
}

// dense linear layer (Tape matmul + bias + gelu_erf), tcgen05
size_t affmae_linear_workspace(int64_t m, int64_t n, int64_t k) { return linear_workspace(m, n, k); }
int affmae_linear_fwd(const affmae_bf16* x, const affmae_bf16* w, const float* bias, int64_t m, int64_t n,
                      int64_t k, int act, affmae_bf16* y, void* workspace, size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return linear_fwd(x, w, bias, m, n, k, act, y, workspace, workspace_bytes, stream);
    )
}

int affmae_linear_fwd_gelu_aux(const affmae_bf16* x, const affmae_bf16* w, const float* bias, int64_t m,
                               int64_t n, int64_t k, affmae_bf16* y, affmae_bf16* pre, void* workspace,
                               size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return linear_fwd_gelu_aux(x, w, bias, m, n, k, y, pre, workspace, workspace_bytes, stream);
    )
}
int affmae_gelu_bwd(const affmae_bf16* pre, const affmae_bf16* dy, int64_t n, affmae_bf16* dpre, void* stream) {
    AFFMAE_GUARD(
        return gelu_bwd(pre, dy, n, dpre, stream);
    )
}
size_t affmae_linear_bwd_workspace(int64_t m, int64_t n, int64_t k) { return linear_bwd_workspace(m, n, k); }
int affmae_linear_bwd(const affmae_bf16* x, const affmae_bf16* w, const affmae_bf16* dy, int64_t m, int64_t n,
                      int64_t k, affmae_bf16* dx, float* dw, float* db, void* workspace, size_t workspace_bytes,
                      void* stream) {
    AFFMAE_GUARD(
        return linear_bwd(x, w, dy, m, n, k, dx, dw, db, workspace, workspace_bytes, stream);
    )
}
int affmae_linear_fwd_add(const affmae_bf16* x, const affmae_bf16* w, const float* bias, int64_t m, int64_t n,
                          int64_t k, const affmae_bf16* c, affmae_bf16* y, void* stream) {
    AFFMAE_GUARD(
        return linear_fwd_add(x, w, bias, m, n, k, c, y, nullptr, 0, stream);
    )
}
int affmae_linear_dx_gelu(const affmae_bf16* dy, const affmae_bf16* w, const affmae_bf16* pre, int64_t m, int64_t n,
                          int64_t k, affmae_bf16* dh, void* stream) {
    AFFMAE_GUARD(
        return linear_dx_gelu(dy, w, pre, m, n, k, dh, stream);
    )
}
int affmae_linear_dx_f32(const affmae_bf16* dy, const affmae_bf16* w, int64_t m, int64_t n, int64_t k, float* dx,
                         float beta, void* stream) {
    AFFMAE_GUARD(
        return linear_dx_f32(dy, w, m, n, k, dx, beta, nullptr, 0, stream);
    )
}

// Tape::layer_norm forward / VJP (proj/src/tape.cpp:84-100,581-617)
int affmae_layernorm_fwd(const affmae_bf16* x, const float* gamma, const float* beta, int64_t rows, int64_t cols,
                         affmae_bf16* y, float* stats, void* stream) {
    AFFMAE_GUARD(
        return layernorm_fwd(x, gamma, beta, rows, cols, y, stats, stream);
    )
}
size_t affmae_layernorm_bwd_workspace(int64_t rows, int64_t cols) { return layernorm_bwd_workspace(rows, cols); }
int affmae_layernorm_bwd(const affmae_bf16* x, const float* gamma, const float* stats, const affmae_bf16* dy,
                         int64_t rows, int64_t cols, affmae_bf16* dx, float* dgamma, float* dbeta, void* workspace,
                         size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return layernorm_bwd(x, gamma, stats, dy, rows, cols, dx, dgamma, dbeta, workspace, workspace_bytes, stream);
    )
}

// NormClampOp (proj/src/pipeline.cpp:75-127) and the masked reconstruction loss (tape.cpp:431-446)
int affmae_norm_clamp_fwd(const affmae_bf16* x, int64_t rows, int64_t d, double limit, affmae_bf16* y, void* stream) {
    AFFMAE_GUARD(
        return norm_clamp_fwd(x, rows, d, limit, y, stream);
    )
}
int affmae_norm_clamp_bwd(const affmae_bf16* x, const affmae_bf16* g, int64_t rows, int64_t d, double limit,
                          affmae_bf16* dx, void* stream) {
    AFFMAE_GUARD(
        return norm_clamp_bwd(x, g, rows, d, limit, dx, stream);
    )
}
size_t affmae_masked_mse_workspace(int64_t rows) { return masked_mse_workspace(rows); }
int affmae_masked_mse(const affmae_bf16* pred, const float* patches, const int32_t* cells, int64_t rows, int64_t p,
                      float* loss, affmae_bf16* dpred, float dloss, void* workspace, size_t workspace_bytes,
                      void* stream) {
    AFFMAE_GUARD(
        return masked_mse(pred, patches, cells, rows, p, loss, dpred, dloss, workspace, workspace_bytes, stream);
    )
}

// AdamW::lr_at / AdamW::step (proj/src/pipeline.cpp:643-680)
double affmae_adamw_lr(const affmae_adamw_cfg* cfg, int64_t step) { return cfg ? adamw_lr(cfg, step) : 0.0; }
int affmae_adamw_step(const affmae_adamw_cfg* cfg, int64_t step, int64_t n_segments, const int64_t* seg_off,
                      const uint8_t* seg_decay, int64_t n, float* value, const float* grad, float* m, float* v,
                      void* stream) {
    AFFMAE_GUARD(
        return adamw_step(cfg, step, n_segments, seg_off, seg_decay, n, value, grad, m, v, stream);
    )
}

// retained_count (proj/src/merging.cpp:50-54)
int64_t affmae_retained_count(int64_t n, double d_s) {
    int64_t r = retained_count_impl(n, d_s);
    if (r < 0) fail(AFFMAE_ECONFIG, "retained_count: d_s must be in (0, 1]");
    return r;
}

size_t affmae_select_retained_workspace(int64_t batch, int64_t tokens) {
    return select_retained_workspace(batch, tokens);
}

int affmae_select_retained(const float* scores, int64_t batch, int64_t tokens, double d_s,
                           int32_t* retained, void* workspace, size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return select_retained(scores, batch, tokens, d_s, retained, workspace, workspace_bytes, stream);
    )
}

size_t affmae_merge_plan_workspace(int64_t batch, int64_t tokens, int64_t retained) {
    return merge_plan_workspace(batch, tokens, retained);
}

int affmae_merge_plan_build(const float* coords, const int32_t* retained, int64_t batch,
                            int64_t tokens, int64_t n_retained, int k_m, affmae_merge_plan* plan,
                            void* workspace, size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return merge_plan_build(coords, retained, batch, tokens, n_retained, k_m, plan, workspace,
                                workspace_bytes, stream);
    )
}

int affmae_importance_scores(const float* feats, int64_t rows, int64_t dim, const float* w1, const float* b1,
                             const float* w2, const float* b2, int hidden, float* scores, void* stream) {
    AFFMAE_GUARD(return importance_scores(feats, rows, dim, w1, b1, w2, b2, hidden, scores, stream);)
}

size_t affmae_merge_tokens_workspace(int64_t batch, int64_t tokens, int64_t n_retained, int64_t dim, int k_m) {
    return merge_tokens_workspace(batch, tokens, n_retained, dim, k_m);
}

int affmae_merge_tokens(const float* coords, const affmae_bf16* feats, const float* scores, const int32_t* retained,
                        int64_t batch, int64_t tokens, int64_t n_retained, int64_t dim, int k_m,
                        const float* p_merge, const affmae_bf16* proj_wt, const float* ln_gamma,
                        const float* ln_beta, affmae_bf16* out_feats, float* out_coords, void* workspace,
                        size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(return merge_tokens(coords, feats, scores, retained, batch, tokens, n_retained, dim, k_m, p_merge,
                                     proj_wt, ln_gamma, ln_beta, out_feats, out_coords, workspace, workspace_bytes,
                                     stream);)
}

int affmae_merge_pool_fwd(const affmae_bf16* feats, const float* scores, const float* p_merge,
                          const int32_t* retained, const affmae_merge_plan* plan, int64_t batch,
                          int64_t tokens, int64_t n_retained, int64_t dim, int k_m,
                          affmae_bf16* out, void* stream) {
    AFFMAE_GUARD(
        return merge_pool_fwd(feats, scores, p_merge, retained, plan, batch, tokens, n_retained, dim,
                              k_m, out, stream);
    )
}

size_t affmae_merge_pool_bwd_workspace(int64_t batch, int64_t n_retained) {
    return merge_pool_bwd_workspace(batch, n_retained);
}

int affmae_merge_pool_bwd(const affmae_bf16* feats, const float* scores, const float* p_merge,
                          const int32_t* retained, const affmae_merge_plan* plan, int64_t batch,
                          int64_t tokens, int64_t n_retained, int64_t dim, int k_m,
                          const affmae_bf16* dout, affmae_bf16* dfeats, float* dscores,
                          float* dp, void* workspace, size_t workspace_bytes, void* stream) {
    AFFMAE_GUARD(
        return merge_pool_bwd(feats, scores, p_merge, retained, plan, batch, tokens, n_retained, dim,
                              k_m, dout, dfeats, dscores, dp, workspace, workspace_bytes, stream);
    )
}

}  // extern "C"
