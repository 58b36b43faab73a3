/*
 * affmae_b200.h — C ABI of the B200-native AFFMAE hot path (libaffmae_b200.so).
 *
 * Plain pointers and sizes only; every call is asynchronous on the caller's
 * CUDA stream (passed as `void*`, a cudaStream_t; NULL = legacy default
 * stream).  All tensor pointers are DEVICE pointers unless a name ends in
 * `_host`.  Batched: B images of N tokens each (the reference is batch-1;
 * exact mask counts make every image in a batch the same size,
 * SURVEY.md §0.9).  Token order inside an image is the reference's order
 * (ascending patch index for stage 0, ascending retained index afterwards).
 *
 * Status codes (reference error taxonomy, proj/include/affmae/errors.hpp:8-15):
 *   AFFMAE_OK 0, AFFMAE_ECONFIG 2 (ConfigError), AFFMAE_ENUMERIC 3
 *   (NumericError), AFFMAE_EUNSUPPORTED 4 (shape outside the compiled kernel
 *   variants; maps to ConfigError), AFFMAE_ECUDA 5 (CUDA runtime failure).
 * affmae_last_error() returns the calling thread's last message.
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to the reference checkout's proj/).
 */
#ifndef AFFMAE_B200_H
#define AFFMAE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFFMAE_OK 0
#define AFFMAE_ECONFIG 2
#define AFFMAE_ENUMERIC 3
#define AFFMAE_EUNSUPPORTED 4
#define AFFMAE_ECUDA 5

typedef uint16_t affmae_bf16; /* IEEE bfloat16 bit pattern */

const char* affmae_last_error(void);
int affmae_version(void);

/* ------------------------------------------------------------------------
 * Cluster geometry (closed forms of balanced_clusters / cluster_neighborhood,
 * src/geometry.cpp:108-131,133-156).  Fill batch/tokens/cluster/groups, call
 * affmae_cluster_geometry to validate and derive the rest.
 * ---------------------------------------------------------------------- */
typedef struct affmae_cluster_geom {
    int64_t batch;      /* B images */
    int64_t tokens;     /* N tokens per image */
    int64_t cluster;    /* requested cluster size (balanced_clusters `size`) */
    int64_t groups;     /* requested neighbour groups (cluster_neighborhood `groups`) */
    /* derived */
    int64_t n_clusters; /* C = ceil(N / min(size, N)) */
    int64_t groups_eff; /* G = min(groups, C) */
    int64_t max_size;   /* ceil(N / C): largest cluster */
    int64_t width;      /* M = G * max_size: NeighborIndex::width */
} affmae_cluster_geom;

int affmae_cluster_geometry(affmae_cluster_geom* g);

/* Device-resident cluster index of one batch.  Cluster k of image b holds
 * curve positions [k*base + min(k,rem), ... + base + (k<rem)) of perm[b],
 * base = N / C, rem = N % C (balanced_clusters, src/geometry.cpp:111-129). */
typedef struct affmae_cluster_index {
    int32_t* perm;       /* [B, N]   sfc_order (src/geometry.cpp:69-106) */
    int32_t* cluster_of; /* [B, N]   ClusterAssignment::cluster_of */
    int32_t* nbr_cl;     /* [B, C, G] own cluster first, then the G-1 nearest
                                      centroids by (d^2, j) (src/geometry.cpp:157-172) */
    int32_t* rev_off;    /* [B, C+1] reverse-neighbour CSR offsets (for attention bwd) */
    int32_t* rev_cl;     /* [B, C*G] query clusters listing cluster c', ascending */
} affmae_cluster_index;

/* Workspace bytes for affmae_cluster_index_build. */
size_t affmae_cluster_index_workspace(const affmae_cluster_geom* g);

/* Replaces balanced_clusters + cluster_neighborhood
 * (include/affmae/geometry.hpp:61-68; src/geometry.cpp:108-186), batched.
 * coords: [B, N, 2] float32 pixel centres.  Bit-exact with the reference. */
int affmae_cluster_index_build(const affmae_cluster_geom* g, const float* coords,
                               affmae_cluster_index* out, void* workspace,
                               size_t workspace_bytes, void* stream);

/* Expands the compact index into the reference's NeighborIndex layout
 * (include/affmae/geometry.hpp:33-48): idx [B, N, M] int32 (padding 0),
 * valid [B, N, M] uint8. For parity dumps and generic consumers. */
int affmae_neighbor_expand(const affmae_cluster_geom* g, const int32_t* perm,
                           const int32_t* nbr_cl, int32_t* idx, uint8_t* valid, void* stream);

/* Replaces sfc_order (src/geometry.cpp:69-106), batched: perm [B, N]. */
size_t affmae_sfc_order_workspace(int64_t batch, int64_t tokens);
int affmae_sfc_order(const float* coords, int64_t batch, int64_t tokens, int32_t* perm,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Replaces knn (src/geometry.cpp:188-216), batched: queries [B, Q, 2],
 * keys [B, K, 2] -> idx [B, Q, k] int32, valid [B, Q, k] uint8.  Exact
 * (d^2 in binary64, ties to the lower key index). */
int affmae_knn(const float* queries, const float* keys, int64_t batch, int64_t n_queries,
               int64_t n_keys, int64_t k, int32_t* idx, uint8_t* valid, void* stream);

/* Replaces make_interp_op (include/affmae/interpolation.hpp:60; InterpOp,
 * src/interpolation.cpp:192-251 over interp_softmax :51-67 / interp_backward
 * :93-142), batched: queries [B, Q, 2], key_coords [B, N, 2], feats [B, N, D]
 * bf16 (D in {64, 128, 256, 512}), neighbour rows idx/valid [B, Q, K] (K <= 32,
 * e.g. from affmae_knn), temperature p (device scalar, a tape parameter),
 * eps (kInterpEps = 1e-6).  out [B, Q, D] bf16 = sum_i softmax(-p d)_i f_i.
 * The backward ACCUMULATES (+=, CustomOp::backward) into dfeats [B, N, D] fp32,
 * dp [1] and dqueries [B, Q, 2]; it needs no workspace.  A row without a valid
 * neighbour yields zeros and no gradient (the reference raises ConfigError). */
int affmae_interp_fwd(const float* queries, const float* key_coords, const affmae_bf16* feats,
                      const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t n_queries,
                      int64_t n_keys, int64_t dim, int64_t k, const float* p, double eps,
                      affmae_bf16* out, void* stream);
int affmae_interp_bwd(const float* queries, const float* key_coords, const affmae_bf16* feats,
                      const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t n_queries,
                      int64_t n_keys, int64_t dim, int64_t k, const float* p, double eps,
                      const affmae_bf16* dout, float* dfeats, float* dp, float* dqueries, void* stream);
/* The same backward with dfeats gathered through a reverse CSR of the rows (key -> the
 * (row, slot) entries naming it, rebuilt per call in the workspace) instead of scattered fp32
 * reductions: each dfeats row is read and written once.  Same semantics and results
 * (to fp32 rounding); batch * n_queries * k < 2^31. */
size_t affmae_interp_bwd_gather_workspace(int64_t batch, int64_t n_queries, int64_t n_keys, int64_t k);
int affmae_interp_bwd_gather(const float* queries, const float* key_coords, const affmae_bf16* feats,
                             const int32_t* idx, const uint8_t* valid, int64_t batch, int64_t n_queries,
                             int64_t n_keys, int64_t dim, int64_t k, const float* p, double eps,
                             const affmae_bf16* dout, float* dfeats, float* dp, float* dqueries,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Row LayerNorm (Tape::layer_norm, src/tape.cpp:84-100, VJP :581-617; eps 1e-5):
 * x, y [rows, cols] bf16, gamma/beta [cols] fp32, stats [rows] float2 {mean, rstd}
 * (written by the forward, read by the backward); cols in {128, 256, 384, 512,
 * 768, 1024}.  The backward overwrites dx (bf16; NULL to skip) and ACCUMULATES
 * dgamma/dbeta (fp32, +=, fixed-order reduction; either may be NULL). */
int affmae_layernorm_fwd(const affmae_bf16* x, const float* gamma, const float* beta, int64_t rows, int64_t cols,
                         affmae_bf16* y, float* stats, void* stream);
size_t affmae_layernorm_bwd_workspace(int64_t rows, int64_t cols);
int affmae_layernorm_bwd(const affmae_bf16* x, const float* gamma, const float* stats, const affmae_bf16* dy,
                         int64_t rows, int64_t cols, affmae_bf16* dx, float* dgamma, float* dbeta, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Decoder row ops (§8(f) #2).  NormClampOp (src/pipeline.cpp:75-127): rows of
 * x [rows, d] bf16 rescaled to norm <= limit; the backward ACCUMULATES into dx (bf16,
 * +=, CustomOp::backward semantics, include/affmae/tape.hpp:29-31).  Reconstruction loss (Tape::mse over the masked cells,
 * src/tape.cpp:431-446, Model::loss_parts src/pipeline.cpp:581-600): loss = mean
 * over rows x p of (pred[r] - patches[cells[r]])^2, pred [rows, p] bf16, patches
 * [n_cells, p] fp32, cells [rows] int32; with dpred != NULL also writes
 * dpred = 2 (pred - target) dloss / numel (bf16).  Deterministic. */
int affmae_norm_clamp_fwd(const affmae_bf16* x, int64_t rows, int64_t d, double limit, affmae_bf16* y, void* stream);
int affmae_norm_clamp_bwd(const affmae_bf16* x, const affmae_bf16* g, int64_t rows, int64_t d, double limit,
                          affmae_bf16* dx, void* stream);
size_t affmae_masked_mse_workspace(int64_t rows);
int affmae_masked_mse(const affmae_bf16* pred, const float* patches, const int32_t* cells, int64_t rows, int64_t p,
                      float* loss, affmae_bf16* dpred, float dloss, void* workspace, size_t workspace_bytes,
                      void* stream);

/* Replaces AdamW (include/affmae/pipeline.hpp:112-127; src/pipeline.cpp:639-680):
 * one optimizer step over every parameter tensor at once.  The tensors live back
 * to back in flat fp32 buffers value/grad/m/v [n] (16-byte aligned; m, v start at
 * zero like the reference's moments); seg_off [n_segments] (DEVICE, ascending
 * start offsets, seg_off[0] = 0) and seg_decay [n_segments] (DEVICE, 1 iff the
 * tensor is a matrix, dim(0) > 1) describe them.  `step` is the number of steps
 * already taken (AdamW::t_): lr_at(step), bias corrections with n = step + 1. */
typedef struct affmae_adamw_cfg {
    double lr;             /* OptimConfig::lr (include/affmae/config.hpp:27-33) */
    int64_t warmup;
    double weight_decay;
    double beta1, beta2;
    int64_t total_steps;   /* AdamW(cfg, total_steps) */
} affmae_adamw_cfg;
double affmae_adamw_lr(const affmae_adamw_cfg* cfg, int64_t step);
int affmae_adamw_step(const affmae_adamw_cfg* cfg, int64_t step, int64_t n_segments, const int64_t* seg_off,
                      const uint8_t* seg_decay, int64_t n, float* value, const float* grad, float* m, float* v,
                      void* stream);

/* Dense linear layer on the tcgen05 tensor cores (the model's QKV / output /
 * MLP / merge projections: Tape matmul + bias (+ gelu_erf), src/tape.cpp,
 * src/pipeline.cpp:388-400,453-458):  y = act(x W^T + b), x [M, K] bf16
 * row-major, W [N, K] bf16 row-major, b [N] fp32, act 0 = identity, 1 = GELU
 * (erf); y [M, N] bf16.  K and N multiples of 8. */
size_t affmae_linear_workspace(int64_t m, int64_t n, int64_t k);
int affmae_linear_fwd(const affmae_bf16* x, const affmae_bf16* w, const float* bias, int64_t m, int64_t n,
                      int64_t k, int act, affmae_bf16* y, void* workspace, size_t workspace_bytes, void* stream);
/* GELU variant that also stores the pre-activation x W^T + b (bf16 [M, N]) for the
 * backward, and the GELU derivative dpre = dy * gelu'(pre) (gelu_bwd, src/tape.cpp;
 * n elements, a multiple of 8). */
int affmae_linear_fwd_gelu_aux(const affmae_bf16* x, const affmae_bf16* w, const float* bias, int64_t m,
                               int64_t n, int64_t k, affmae_bf16* y, affmae_bf16* pre, void* workspace,
                               size_t workspace_bytes, void* stream);
int affmae_gelu_bwd(const affmae_bf16* pre, const affmae_bf16* dy, int64_t n, affmae_bf16* dpre, void* stream);
/* Backward of y = x W^T + b given dy (already through the activation): dx [M, K] bf16
 * (overwritten), dw [N, K] fp32 and db [N] fp32 ACCUMULATED (+=); any output may be NULL.
 * M, N, K multiples of 8. */
size_t affmae_linear_bwd_workspace(int64_t m, int64_t n, int64_t k);
int affmae_linear_bwd(const affmae_bf16* x, const affmae_bf16* w, const affmae_bf16* dy, int64_t m, int64_t n,
                      int64_t k, affmae_bf16* dx, float* dw, float* db, void* workspace, size_t workspace_bytes,
                      void* stream);
/* Fused variants of the block's layers (the training step's GEMM epilogues):
 *   affmae_linear_fwd_add:  y = x W^T + b + c   (c bf16 [M, N], the residual, summed in fp32)
 *   affmae_linear_dx_gelu:  dh = (dy W) * gelu'(pre)   (dy [M, N], pre / dh bf16 [M, K]):
 *                           linear_bwd's dX and gelu_bwd in one pass
 *   affmae_linear_dx_f32:   dx = dy W + beta * dx   (dx fp32 [M, K]; beta 0 overwrites) */
int affmae_linear_fwd_add(const affmae_bf16* x, const affmae_bf16* w, const float* bias, int64_t m, int64_t n,
                          int64_t k, const affmae_bf16* c, affmae_bf16* y, void* stream);
int affmae_linear_dx_gelu(const affmae_bf16* dy, const affmae_bf16* w, const affmae_bf16* pre, int64_t m, int64_t n,
                          int64_t k, affmae_bf16* dh, void* stream);
int affmae_linear_dx_f32(const affmae_bf16* dy, const affmae_bf16* w, int64_t m, int64_t n, int64_t k, float* dx,
                         float beta, void* stream);

/* ------------------------------------------------------------------------
 * Cluster attention (nbhd_attn_streaming / nbhd_attn_backward,
 * include/affmae/attention.hpp:52-72; AttnOp, src/attention.cpp:374-444).
 * ---------------------------------------------------------------------- */
typedef struct affmae_attn_desc {
    int heads;
    int head_dim;
    int bias_hidden; /* BiasNet hidden width H */
    double patch;    /* BiasNet offset normaliser */
} affmae_attn_desc;

typedef struct affmae_attn_inputs {
    const affmae_bf16* q;       /* [B, N, heads*head_dim] */
    const affmae_bf16* k;       /* [B, N, heads*head_dim] */
    const affmae_bf16* v;       /* [B, N, heads*head_dim] */
    const affmae_bf16* blank_k; /* [heads, head_dim] */
    const affmae_bf16* blank_v; /* [heads, head_dim] */
    const float* coords;        /* [B, N, 2] */
    const float* w1;            /* [heads, 2H]  BiasNet (include/affmae/attention.hpp:16-29) */
    const float* b1;            /* [heads, H] */
    const float* w2;            /* [heads, H] */
    const float* b2;            /* [heads] */
    const float* blank;         /* [heads]  blank-slot bias */
} affmae_attn_inputs;

/* Workspace bytes for affmae_attn_fwd (holds the per-call BiasNet offset table). */
size_t affmae_attn_fwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a);

/* Forward: out [B, N, heads*head_dim] bf16 and lse [B, N, heads] fp32
 * (natural-log softmax normaliser, kept for the backward). */
int affmae_attn_fwd(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                    const affmae_attn_inputs* in, const int32_t* perm, const int32_t* nbr_cl,
                    affmae_bf16* out, float* lse, void* workspace, size_t workspace_bytes,
                    void* stream);

/* Attention plan: the geometry part of the op (query-cluster records, key /
 * reverse-pair records, lattice classes), built once per cluster index and
 * reused by every forward / backward on it -- the reference's AttnOp freezes
 * coords + NeighborIndex at construction (src/attention.cpp:374-383).  The
 * caller owns `buf` (device, affmae_attn_plan_workspace bytes); build fills
 * the descriptor fields, the planned calls check them. */
typedef struct affmae_attn_plan {
    void* buf;
    size_t bytes;
    int64_t batch, tokens, n_clusters, groups_eff, width; /* filled by build */
    double patch;
    int has_reverse; /* built with the reverse CSR (required by the backward) */
} affmae_attn_plan;

size_t affmae_attn_plan_workspace(const affmae_cluster_geom* g, int with_reverse);
int affmae_attn_plan_build(const affmae_cluster_geom* g, const affmae_attn_desc* a, const float* coords,
                           const affmae_cluster_index* idx, int with_reverse, affmae_attn_plan* plan,
                           void* stream);
/* Per-call workspace of the planned entry points (BiasNet offset table, backward partials). */
size_t affmae_attn_fwd_planned_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a);
int affmae_attn_fwd_planned(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                            const affmae_attn_inputs* in, const affmae_attn_plan* plan, affmae_bf16* out,
                            float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* hilbert_index (include/affmae/geometry.hpp:51; src/geometry.cpp:15-30), host side */
uint64_t affmae_hilbert_index(uint32_t n, uint32_t x, uint32_t y);

/* flop_count_attn / flop_count_attn_dense (include/affmae/attention.hpp:77-79,
 * src/attention.cpp:360-370): closed-form forward flops of neighbourhood attention,
 * 4 n (m+1) h d + 6 n (m+1) h, and of dense attention, 4 n^2 h d + 6 n^2 h.  Returns 0
 * (and sets ConfigError's message) when an argument is not positive. */
uint64_t affmae_flop_count_attn(int64_t n, int64_t m, int64_t h, int64_t d);
uint64_t affmae_flop_count_attn_dense(int64_t n, int64_t h, int64_t d);

typedef struct affmae_attn_grads {
    affmae_bf16* dq;  /* [B, N, h*d]  overwritten */
    affmae_bf16* dk;  /* [B, N, h*d]  overwritten */
    affmae_bf16* dv;  /* [B, N, h*d]  overwritten */
    float* dblank_k;  /* [h, d]   accumulated (+=), CustomOp::backward semantics */
    float* dblank_v;  /* [h, d]   += */
    float* dw1;       /* [h, 2H]  += */
    float* db1;       /* [h, H]   += */
    float* dw2;       /* [h, H]   += */
    float* db2;       /* [h]      += */
    float* dblank;    /* [h]      += */
} affmae_attn_grads;

size_t affmae_attn_bwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a);

int affmae_attn_bwd(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                    const affmae_attn_inputs* in, const affmae_cluster_index* idx,
                    const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                    affmae_attn_grads* grads, void* workspace, size_t workspace_bytes,
                    void* stream);

size_t affmae_attn_bwd_planned_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a);
int affmae_attn_bwd_planned(const affmae_cluster_geom* g, const affmae_attn_desc* a,
                            const affmae_attn_inputs* in, const affmae_attn_plan* plan,
                            const affmae_bf16* out, const float* lse, const affmae_bf16* dout,
                            affmae_attn_grads* grads, void* workspace, size_t workspace_bytes,
                            void* stream);

/* Attention over arbitrary neighbour rows: nbhd_attn_streaming / nbhd_attn_backward
 * (include/affmae/attention.hpp:52-72) on a general NeighborIndex -- the decoder's
 * cross attention over one_to_one rows and self attention over knn rows
 * (src/pipeline.cpp:64-71, 495-535; attn_layer :467-477).  idx / valid [B, N, width]
 * (width in [1, 31], image-local ids into the same N tokens, e.g. from affmae_knn);
 * head_dim 16, 32 or 64.  Forward: out [B, N, h*d] bf16, lse [B, N, h] fp32.
 * Backward: dq [B, N, h*d] bf16 overwritten; dk, dv [B, N, h*d] fp32 and the
 * parameter gradients ACCUMULATED (+=). */
int affmae_gattn_fwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx,
                     const uint8_t* valid, int64_t batch, int64_t tokens, int64_t width,
                     affmae_bf16* out, float* lse, void* stream);
int affmae_gattn_bwd(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx,
                     const uint8_t* valid, int64_t batch, int64_t tokens, int64_t width,
                     const affmae_bf16* dout, affmae_bf16* dq, float* dk, float* dv,
                     float* dblank_k, float* dblank_v, float* dw1, float* db1, float* dw2,
                     float* db2, float* dblank, void* workspace, size_t workspace_bytes,
                     void* stream);
/* Workspace for the gather-mode backward (0 if heads*head_dim is not 32..512, power of two).
 * With a workspace, dk / dv are gathered over a per-call reverse CSR of the rows (key -> the
 * (row, slot) entries naming it) instead of scattered fp32 reductions; NULL = scatter mode. */
size_t affmae_gattn_bwd_workspace(const affmae_attn_desc* a, int64_t batch, int64_t tokens, int64_t width);

/* ------------------------------------------------------------------------
 * Inputs on the device.
 * ---------------------------------------------------------------------- */
/* Replaces perlin_field + mask_from_field (include/affmae/masking.hpp; src/masking.cpp:34-92),
 * batched: seeds_host [B] (HOST array, the per-image MaskSpec seeds), grid h x w, octaves /
 * base_freq / persistence as perlin_field, ratio as mask_from_field -> masked [B, h, w] uint8
 * (1 = hidden), exactly llround(ratio*h*w) per image, largest field first, ties to the lower
 * cell.  Bit-exact with the reference (the corner gradients are computed on the host). */
size_t affmae_perlin_mask_workspace(int64_t batch, int64_t h, int64_t w, int octaves, double base_freq);
int affmae_perlin_mask(const uint64_t* seeds_host, int64_t batch, int64_t h, int64_t w, int octaves,
                       double base_freq, double persistence, double ratio, uint8_t* masked,
                       void* workspace, size_t workspace_bytes, void* stream);
/* Stage-0 coordinates of the visible cells in ascending cell index (src/geometry.cpp:44-50,
 * src/pipeline.cpp:412-427): coords [B, nvis, 2] float32 pixel centres c*patch + patch/2;
 * count [B] (optional) receives each image's visible count; rows beyond nvis are dropped. */
int affmae_visible_coords(const uint8_t* masked, int64_t batch, int64_t h, int64_t w, double patch,
                          int64_t nvis, float* coords, int32_t* count, void* stream);
/* Replaces synth_image (src/pipeline.cpp:169-227), batched: img [B, size, size] float64 for
 * seeds_host [B].  Matches the reference to ~1e-15 (device exp() is within 1 ulp of glibc's);
 * synchronises `stream` before returning (the per-image draws are staged from the host). */
/* patchify (src/pipeline.cpp:131-150): img [B, h, w] float64 -> vectors [B, (h/p)*(w/p), p*p]
 * float32 row-major patches.  affmae_masked_rows: the masked cells of each image in ascending
 * index as global rows b*cells + cell -> rows [B, nmask] (Model::loss_parts target rows,
 * src/pipeline.cpp:588-596; the `cells` argument of affmae_masked_mse). */
int affmae_patchify(const double* img, int64_t batch, int64_t h, int64_t w, int64_t patch, float* vectors,
                    void* stream);
int affmae_masked_rows(const uint8_t* masked, int64_t batch, int64_t cells, int64_t nmask, int32_t* rows,
                       void* stream);
size_t affmae_synth_images_workspace(int64_t batch, int64_t size);
int affmae_synth_images(const uint64_t* seeds_host, int64_t batch, int64_t size, double* img, void* workspace,
                        size_t workspace_bytes, void* stream);

/* AFT1 tensor files (write_aft / read_aft, src/tensor_io.cpp:60-105; format
 * include/affmae/tensor_io.hpp:11-13) from / into DEVICE buffers.  write: dev_src holds fp32
 * values (dtype 0 = b32, 1 = b16emu) or bytes (dtype 2); the file is byte-identical to the
 * reference's for the same values.  read: fp32 values (u8 payloads as byte values) into
 * dev_dst[capacity]; *numel_out (optional) gets the element count.  Both synchronise `stream`. */
int affmae_aft_write(const char* path, const void* dev_src, const int64_t* dims, int ndim, int dtype,
                     void* stream);
int affmae_aft_read_header(const char* path, int* dtype, int* ndim, int64_t* dims /* [8] */);
int affmae_aft_read(const char* path, float* dev_dst, int64_t capacity, int64_t* numel_out, void* stream);
/* save_checkpoint / load_checkpoint (src/pipeline.cpp:757-797) over device fp32 parameter
 * buffers: <dir>/<name>.aft per parameter + manifest.tsv ("name\td0xd1\tprec\tfile"), prec
 * codes 0 b32 / 1 b16emu / 2 b64 (stored as b32).  load: unknown, missing or mis-sized
 * parameters are ConfigErrors, as in the reference. */
int affmae_checkpoint_save(const char* dir, int n, const char* const* names, const float* const* dev_vals,
                           const int64_t* const* dims, const int* ndims, const int* precs, void* stream);
int affmae_checkpoint_load(const char* dir, int n, const char* const* names, float* const* dev_vals,
                           const int64_t* numels, void* stream);

/* ------------------------------------------------------------------------
 * Adaptive KNN merge (src/merging.cpp).
 * ---------------------------------------------------------------------- */

/* retained_count (src/merging.cpp:50-54); -2 on d_s outside (0, 1]. */
int64_t affmae_retained_count(int64_t n, double d_s);

size_t affmae_select_retained_workspace(int64_t batch, int64_t tokens);
/* select_retained (src/merging.cpp:56-69), batched: scores [B, N] fp32 ->
 * retained [B, R] int32 ascending, R = retained_count(N, d_s).  Bit-exact. */
int affmae_select_retained(const float* scores, int64_t batch, int64_t tokens, double d_s,
                           int32_t* retained, void* workspace, size_t workspace_bytes,
                           void* stream);

typedef struct affmae_merge_plan {
    int32_t* target;    /* [B, N]  retained index each dropped token goes to; -1 for retained */
    int32_t* pool_idx;  /* [B, R, k_m] contributor token indices, (dist, index) ascending */
    double* pool_dist;  /* [B, R, k_m] Euclidean distances (binary64, bit-exact) */
    int32_t* pool_cnt;  /* [B, R] valid entries per pool (<= k_m) */
    int32_t* row_of;    /* [B, N]  output row a token feeds: retained -> its own row, pooled
                                   dropped -> its pool's row, truncated dropped -> -1 */
} affmae_merge_plan;

size_t affmae_merge_plan_workspace(int64_t batch, int64_t tokens, int64_t retained);
/* merge_plan (src/merging.cpp:71-116), batched; coords [B, N, 2],
 * retained [B, R] ascending.  Bit-exact (first-minimum tie rule). */
int affmae_merge_plan_build(const float* coords, const int32_t* retained, int64_t batch,
                            int64_t tokens, int64_t n_retained, int k_m, affmae_merge_plan* plan,
                            void* workspace, size_t workspace_bytes, void* stream);

/* MergePoolOp::forward (src/merging.cpp:121-166): out [B, R, 2D] bf16 rows
 * [f_r ; sum_t softmax(-p*dist)_t * s_j * f_j].  p_merge is a device scalar. */
int affmae_merge_pool_fwd(const affmae_bf16* feats, const float* scores, const float* p_merge,
                          const int32_t* retained, const affmae_merge_plan* plan, int64_t batch,
                          int64_t tokens, int64_t n_retained, int64_t dim, int k_m,
                          affmae_bf16* out, void* stream);

/* importance_scores (src/merging.cpp:31-48): scores[i] = sigmoid(GELU(f_i W1 + b1) w2 + b2)
 * for feats [rows, dim] fp32, W1 [dim, hidden] (the reference's MergeParams layout), b1
 * [hidden], w2 [hidden], b2 [1], hidden <= 32; binary64 in the reference's operation order,
 * rounded once to fp32 (equal to the reference's b32 output up to the device erf / exp's
 * last binary64 bit). */
int affmae_importance_scores(const float* feats, int64_t rows, int64_t dim, const float* w1, const float* b1,
                             const float* w2, const float* b2, int hidden, float* scores, void* stream);

/* merge_tokens (src/merging.cpp:242-273), batched: per image, the merge plan of `retained`
 * (bit-exact), the pool rows [f_r ; agg], the [2D -> D] projection on the tensor cores and
 * layer_norm_rows (eps 1e-5).  feats [B, N, D] bf16, coords [B, N, 2], scores [B, N],
 * retained [B, R] ascending, proj_wt [D, 2D] bf16 = the reference's proj_w [2D, D]
 * transposed, ln_gamma / ln_beta [D] fp32, p_merge a device scalar.  Outputs: merged
 * feats [B, R, D] bf16, the retained coords [B, R, 2].  D a multiple of 64 up to 1024. */
size_t affmae_merge_tokens_workspace(int64_t batch, int64_t tokens, int64_t n_retained, int64_t dim, int k_m);
int affmae_merge_tokens(const float* coords, const affmae_bf16* feats, const float* scores, const int32_t* retained,
                        int64_t batch, int64_t tokens, int64_t n_retained, int64_t dim, int k_m,
                        const float* p_merge, const affmae_bf16* proj_wt, const float* ln_gamma,
                        const float* ln_beta, affmae_bf16* out_feats, float* out_coords, void* workspace,
                        size_t workspace_bytes, void* stream);

size_t affmae_merge_pool_bwd_workspace(int64_t batch, int64_t n_retained);
/* MergePoolOp::backward (src/merging.cpp:169-219): dfeats [B, N, D] bf16 and
 * dscores [B, N] fp32 are overwritten (every token receives at most one
 * contribution); dp [1] fp32 is accumulated (+=). */
int affmae_merge_pool_bwd(const affmae_bf16* feats, const float* scores, const float* p_merge,
                          const int32_t* retained, const affmae_merge_plan* plan, int64_t batch,
                          int64_t tokens, int64_t n_retained, int64_t dim, int k_m,
                          const affmae_bf16* dout, affmae_bf16* dfeats, float* dscores,
                          float* dp, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Device-resident training step (SURVEY.md §8(a) Model::encode stage loop, §8(f) #1-#3):
 * Model::encode / decode / deep_sup / loss_parts (src/pipeline.cpp:402-610), the Tape's
 * reverse sweep over them (src/tape.cpp:466-724) and AdamW (src/pipeline.cpp:639-680) over a
 * batch of images, every op on this library's kernels.  Parameters are fp32 masters (the
 * reference's b32 tape) with bf16 shadows for the tensor-core GEMMs; activations bf16 with an
 * fp32 residual stream.  Batched semantics: the loss is the mean over the batch of the
 * reference's per-image loss, so B = 1 is the reference's step.
 * ---------------------------------------------------------------------- */
typedef struct affmae_stage_cfg {   /* StageConfig (include/affmae/config.hpp:9-17) */
    int64_t dim;
    int heads;
    int blocks;
    int64_t cluster;
    int groups;
    double d_s;
    int interp_k;
} affmae_stage_cfg;

#define AFFMAE_MAX_STAGES 8
typedef struct affmae_model_cfg {   /* PipelineConfig (include/affmae/config.hpp:35-52) */
    int64_t image, patch;
    int n_stages;
    affmae_stage_cfg stages[AFFMAE_MAX_STAGES];
    int64_t dec_dim;                /* DecoderConfig */
    int dec_depth, dec_heads, gather_k, self_k;
    double lambda_aux;
    int mask_strategy;              /* 0 = "perlin", 1 = "random" */
    double mask_ratio;
    affmae_adamw_cfg optim;         /* OptimConfig + the trainer's total step count */
    uint64_t seed;
    int bias_hidden, scorer_hidden, merge_k;
    int64_t batch;                  /* images per step on this device */
} affmae_model_cfg;

typedef struct affmae_model affmae_model;   /* opaque: parameters, optimizer state, activations */

typedef struct affmae_model_info {
    int n_params;          /* parameter tensors (ParamStore order) */
    int64_t n_values;      /* their total element count */
    int64_t tokens[AFFMAE_MAX_STAGES];  /* visible tokens per image entering each stage */
    int64_t masked;        /* masked cells per image (decoder queries) */
    int64_t device_bytes;  /* device memory held by the model */
    int64_t steps_taken;   /* AdamW::steps_taken */
} affmae_model_info;

/* Model(cfg) (src/pipeline.cpp:255-371): validates (ConfigError cases of
 * PipelineConfig::validate, src/config.cpp:37-66, plus the compiled kernel variants) and
 * initialises the parameters exactly as the reference (same splitmix64 draws, fp32). */
int affmae_model_create(const affmae_model_cfg* cfg, affmae_model** out);
void affmae_model_destroy(affmae_model* m);
int affmae_model_get_info(const affmae_model* m, affmae_model_info* info);
/* parameter i: reference name and dims (rows x cols, the reference's layout) */
const char* affmae_model_param_name(const affmae_model* m, int i);
int affmae_model_param_dims(const affmae_model* m, int i, int64_t* rows, int64_t* cols);
/* all parameters (or their gradients) concatenated in ParamStore order, reference layout,
 * HOST fp32 buffers of n_values (synchronous) */
int affmae_model_get_params(affmae_model* m, float* host);
int affmae_model_set_params(affmae_model* m, const float* host);
int affmae_model_get_grads(affmae_model* m, float* host);
/* Model-owned device input buffers (stable addresses, so a captured step graph can replay):
 * images [B, image, image] float64 (synth_image layout), masked [B, g, g] uint8 (1 = hidden). */
int affmae_model_inputs(affmae_model* m, double** images, uint8_t** masked);
/* Model::make_mask (src/pipeline.cpp:625-637) of B images from seeds_host [B] into the
 * model's mask buffer (perlin: device kernel, bit-exact; random: host shuffle). */
int affmae_model_make_masks(affmae_model* m, const uint64_t* seeds_host, void* stream);
/* zero_grads + encode + decode + deep_sup + loss_parts + Tape::backward on the model's
 * input buffers; gradients of the batch-mean loss left in the model.  loss3 (device fp32
 * [3] or NULL) receives {total, main, aux}. */
int affmae_model_forward_backward(affmae_model* m, float* loss3, void* stream);
/* encode + decode + deep_sup + loss_parts only (masked_mse, src/pipeline.cpp:748-755): loss3 as above */
int affmae_model_forward(affmae_model* m, float* loss3, void* stream);
/* a fresh AdamW(cfg.optim, total_steps) as train() constructs per call (src/pipeline.cpp:686):
 * zero moments, step 0 */
int affmae_model_reset_optimizer(affmae_model* m, int64_t total_steps);
/* AdamW::step over every parameter (src/pipeline.cpp:650-680) + bf16 shadow refresh */
int affmae_model_apply_step(affmae_model* m, void* stream);
/* forward_backward + apply_step; with use_graph the whole step is captured into a CUDA
 * graph on the first call and replayed afterwards */
int affmae_model_train_step(affmae_model* m, float* loss3, int use_graph, void* stream);
/* after forward_backward: stage s's entering coordinates [B, N_s, 2], its features before
 * the merge (EncodeStage::coords / ::feats, include/affmae/pipeline.hpp:57-62) [B, N_s, D_s]
 * and its merge scores [B, N_s] (stages with a merge), copied to HOST fp32 buffers
 * (synchronous; any pointer may be NULL) */
int affmae_model_stage_output(affmae_model* m, int stage, float* coords_host, float* feats_host,
                              float* scores_host);
/* Parity-test hook (teacher forcing): stage s's merge uses retained_host [B, R_s] (ascending
 * token indices, e.g. the reference's retained set) instead of select_retained on the device
 * scores; NULL restores the model's own selection.  Everything else is unchanged. */
int affmae_model_force_retained(affmae_model* m, int stage, const int32_t* retained_host);
/* Data parallelism: images shard over `world` ranks (one process per GPU).
 * The loss gradient is seeded with 1/world, so the SUM of the ranks' gradients is the gradient
 * of the global batch mean.  nccl_id (from affmae_nccl_unique_id on rank 0, broadcast by the
 * caller) makes every forward_backward end with an ncclAllReduce(sum) of the gradient arena
 * on the model's stream (inside the step's graph); NULL leaves the sum to the caller (e.g. a
 * host-staged gloo all-reduce between forward_backward and apply_step). */
int affmae_nccl_unique_id(uint8_t* out128);
int affmae_model_set_world(affmae_model* m, int world, int rank, const uint8_t* nccl_id);
/* flat fp32 gradient arena on the device (for the data-parallel all-reduce between
 * forward_backward and apply_step) */
int affmae_model_grad_buffer(affmae_model* m, float** grad, int64_t* n);
/* save_checkpoint / load_checkpoint (src/pipeline.cpp:757-797): <dir>/manifest.tsv holds
 * the parameters only (the reference loads it unchanged); the AdamW moments and step go to
 * <dir>/optim/ (absent -> the optimizer restarts). */
int affmae_model_save(affmae_model* m, const char* dir);
int affmae_model_load(affmae_model* m, const char* dir);

#ifdef __cplusplus
}
#endif
#endif /* AFFMAE_B200_H */
