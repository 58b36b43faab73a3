// Internal C++ entry points of the kernel translation units (the extern "C" wrappers in
// capi.cu and the model runtime in model.cu call these directly).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "affmae_b200.h"

namespace affmae_b200 {

// implemented in attention.cu / index.cu / merge.cu
size_t attn_fwd_workspace(const affmae_cluster_geom*, const affmae_attn_desc*);
size_t attn_bwd_workspace(const affmae_cluster_geom*, const affmae_attn_desc*);
int attn_fwd(const affmae_cluster_geom*, const affmae_attn_desc*, const affmae_attn_inputs*,
             const int32_t*, const int32_t*, affmae_bf16*, float*, void*, size_t, void*);
int attn_bwd(const affmae_cluster_geom*, const affmae_attn_desc*, const affmae_attn_inputs*,
             const affmae_cluster_index*, const affmae_bf16*, const float*, const affmae_bf16*,
             affmae_attn_grads*, void*, size_t, void*);
size_t attn_plan_workspace(const affmae_cluster_geom*, int);
int attn_plan_build(const affmae_cluster_geom*, const affmae_attn_desc*, const float*,
                    const affmae_cluster_index*, int, affmae_attn_plan*, void*);
size_t attn_fwd_planned_workspace(const affmae_cluster_geom*, const affmae_attn_desc*);
size_t attn_bwd_planned_workspace(const affmae_cluster_geom*, const affmae_attn_desc*);
// ldq: elements between token rows of q/k/v (and dq/dk/dv), 0 = heads*head_dim (an
// interleaved [N, 3D] QKV buffer passes 3*heads*head_dim)
int attn_fwd_planned(const affmae_cluster_geom*, const affmae_attn_desc*, const affmae_attn_inputs*,
                     const affmae_attn_plan*, affmae_bf16*, float*, void*, size_t, void*, int64_t ldq = 0);
int attn_bwd_planned(const affmae_cluster_geom*, const affmae_attn_desc*, const affmae_attn_inputs*,
                     const affmae_attn_plan*, const affmae_bf16*, const float*, const affmae_bf16*,
                     affmae_attn_grads*, void*, size_t, void*, int64_t ldq = 0);
size_t cluster_index_workspace(const affmae_cluster_geom*);
int cluster_index_build(const affmae_cluster_geom*, const float*, affmae_cluster_index*, void*,
                        size_t, void*);
size_t sfc_order_workspace(int64_t, int64_t);
int sfc_order(const float*, int64_t, int64_t, int32_t*, void*, size_t, void*);
int neighbor_expand(const affmae_cluster_geom*, const int32_t*, const int32_t*, int32_t*, uint8_t*,
                    void*);
int knn(const float*, const float*, int64_t, int64_t, int64_t, int64_t, int32_t*, uint8_t*, void*);
int interp_fwd(const float*, const float*, const void*, const int32_t*, const uint8_t*, int64_t, int64_t, int64_t,
               int64_t, int64_t, const float*, double, void*, void*);
int interp_bwd(const float*, const float*, const void*, const int32_t*, const uint8_t*, int64_t, int64_t, int64_t,
               int64_t, int64_t, const float*, double, const void*, float*, float*, float*, void*);
// trailing strides (elements, 0 = dense): q rows, k / v rows, dq rows (see GAttnP)
int gattn_fwd(const affmae_attn_desc*, const affmae_attn_inputs*, const int32_t*, const uint8_t*, int64_t, int64_t,
              int64_t, void*, float*, void*, int64_t ldq = 0, int64_t ldkv = 0);
int gattn_bwd(const affmae_attn_desc*, const affmae_attn_inputs*, const int32_t*, const uint8_t*, int64_t, int64_t,
              int64_t, const void*, void*, float*, float*, float*, float*, float*, float*, float*, float*, float*,
              void*, size_t, void*, int64_t ldq = 0, int64_t ldkv = 0, int64_t ldd = 0);
size_t gattn_bwd_workspace(const affmae_attn_desc*, int64_t, int64_t, int64_t);
// one-to-one rows (idx[i] = i, all valid: the decoder's cross attention): bf16 dk / dv stored
// directly, every row written (no zero fill, reductions or cast pass)
int gattn_bwd_o2o(const affmae_attn_desc* a, const affmae_attn_inputs* in, const int32_t* idx, const uint8_t* valid,
                  int64_t batch, int64_t tokens, const void* dout, void* dq, void* dk_bf16, void* dv_bf16, float* dbk,
                  float* dbv, float* dw1, float* db1, float* dw2, float* db2, float* dblank, void* workspace,
                  size_t ws_bytes, void* stream, int64_t ldq = 0, int64_t ldkv = 0, int64_t ldd = 0,
                  int64_t lddkv = 0);
size_t interp_bwd_gather_workspace(int64_t, int64_t, int64_t, int64_t);
int interp_bwd_gather(const float*, const float*, const void*, const int32_t*, const uint8_t*, int64_t, int64_t,
                      int64_t, int64_t, int64_t, const float*, double, const void*, float*, float*, float*, void*,
                      size_t, void*);
size_t perlin_mask_workspace(int64_t, int64_t, int64_t, int, double);
int perlin_mask(const uint64_t*, int64_t, int64_t, int64_t, int, double, double, double, uint8_t*, void*, size_t,
                void*);
int visible_coords(const uint8_t*, int64_t, int64_t, int64_t, double, int64_t, float*, int32_t*, void*);
int aft_write(const char*, const void*, const int64_t*, int, int, void*);
int aft_read_header(const char*, int*, int*, int64_t*);
int aft_read(const char*, float*, int64_t, int64_t*, void*);
int checkpoint_save(const char*, int, const char* const*, const float* const*, const int64_t* const*, const int*,
                    const int*, void*);
int checkpoint_load(const char*, int, const char* const*, float* const*, const int64_t*, void*);
size_t synth_images_workspace(int64_t, int64_t);
int synth_images(const uint64_t*, int64_t, int64_t, double*, void*, size_t, void*);
int patchify(const double*, int64_t, int64_t, int64_t, int64_t, float*, void*);
int masked_rows(const uint8_t*, int64_t, int64_t, int64_t, int32_t*, void*);
int64_t retained_count_impl(int64_t, double);
double adamw_lr(const affmae_adamw_cfg*, int64_t);
size_t linear_workspace(int64_t, int64_t, int64_t);
int linear_fwd(const void*, const void*, const float*, int64_t, int64_t, int64_t, int, void*, void*, size_t, void*);
size_t linear_bwd_workspace(int64_t, int64_t, int64_t);
int linear_fwd_gelu_aux(const void*, const void*, const float*, int64_t, int64_t, int64_t, void*, void*, void*, size_t,
                        void*);
int gelu_bwd(const void*, const void*, int64_t, void*, void*);
int layernorm_fwd(const void*, const float*, const float*, int64_t, int64_t, void*, float*, void*);
size_t layernorm_bwd_workspace(int64_t, int64_t);
int norm_clamp_fwd(const void*, int64_t, int64_t, double, void*, void*);
int norm_clamp_bwd(const void*, const void*, int64_t, int64_t, double, void*, void*);
size_t masked_mse_workspace(int64_t);
int masked_mse(const void*, const float*, const int32_t*, int64_t, int64_t, float*, void*, float, void*, size_t, void*);
int layernorm_bwd(const void*, const float*, const float*, const void*, int64_t, int64_t, void*, float*, float*, void*,
                  size_t, void*);
int linear_bwd(const void*, const void*, const void*, int64_t, int64_t, int64_t, void*, float*, float*, void*, size_t,
               void*);
int adamw_step(const affmae_adamw_cfg*, int64_t, int64_t, const int64_t*, const uint8_t*, int64_t, float*, const float*,
               float*, float*, void*);
size_t select_retained_workspace(int64_t, int64_t);
int select_retained(const float*, int64_t, int64_t, double, int32_t*, void*, size_t, void*);
size_t merge_plan_workspace(int64_t, int64_t, int64_t);
int importance_scores(const float* feats, int64_t rows, int64_t dim, const float* w1, const float* b1,
                      const float* w2, const float* b2, int hidden, float* out, void* stream);
size_t merge_tokens_workspace(int64_t batch, int64_t n, int64_t r, int64_t dim, int k_m);
int merge_tokens(const float* coords, const void* feats, const float* scores, const int32_t* retained, int64_t batch,
                 int64_t n, int64_t r, int64_t dim, int k_m, const float* p_merge, const void* proj_wt,
                 const float* gamma, const float* beta, void* out_feats, float* out_coords, void* workspace,
                 size_t ws_bytes, void* stream);
int merge_plan_build(const float*, const int32_t*, int64_t, int64_t, int64_t, int, affmae_merge_plan*,
                     void*, size_t, void*);
int merge_pool_fwd(const affmae_bf16*, const float*, const float*, const int32_t*,
                   const affmae_merge_plan*, int64_t, int64_t, int64_t, int64_t, int, affmae_bf16*,
                   void*);
size_t merge_pool_bwd_workspace(int64_t, int64_t);
int merge_pool_bwd(const affmae_bf16*, const float*, const float*, const int32_t*,
                   const affmae_merge_plan*, int64_t, int64_t, int64_t, int64_t, int,
                   const affmae_bf16*, affmae_bf16*, float*, float*, void*, size_t, void*);


// index.cu: hilbert_index (proj/src/geometry.cpp:15-30) on the host
uint64_t hilbert_index_host(uint32_t n, uint32_t x, uint32_t y);
// dist.cu: NCCL loaded at run time (no link-time dependency)
int nccl_unique_id(uint8_t* out128);
int nccl_comm_init(const uint8_t* id128, int nranks, int rank, void** comm);
int nccl_allreduce_sum_f32(void* comm, float* buf, int64_t n, cudaStream_t st);
void nccl_comm_destroy(void* comm);
// optim.cu: AdamW with the step count on the device (advanced by the call) and the bf16
// shadow of the first n_shadow values refreshed in the same pass
int adamw_step_dev(const affmae_adamw_cfg* c, int64_t* step_dev, void* scalars_dev, int64_t n_segments,
                   const int64_t* seg_off, const uint8_t* seg_decay, int64_t n, float* value, const float* grad,
                   float* m, float* v, void* shadow, int64_t n_shadow, void* stream);
size_t adamw_scalars_bytes();
// gemm.cu: y = x W^T + b + c (c bf16 [M, N] added before the rounding)
int linear_fwd_add(const void* x, const void* w, const float* bias, int64_t m, int64_t n, int64_t k, const void* c,
                   void* y, void* ws, size_t ws_bytes, void* stream);
// gemm.cu: dH = (dY W) * GELU'(pre) (bf16), the MLP's fc2 input gradient with the
// activation derivative fused into the GEMM epilogue
int linear_dx_gelu(const void* dy, const void* w, const void* pre, int64_t m, int64_t n, int64_t k, void* dh,
                   void* stream);
// gemm.cu: dX = dY W into fp32 with D = dY W + beta * D (beta 0 overwrites, 1 accumulates)
int linear_dx_f32(const void* dy, const void* w, int64_t m, int64_t n, int64_t k, float* dx, float beta, void* ws,
                  size_t ws_bytes, void* stream);

}  // namespace affmae_b200
