/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so; it is the checker, never the thing measured or shipped.
 * Every function restates the reference algorithm with the same arithmetic
 * order (so results are bit-identical to the reference's own build, which the
 * CPU test-suite verifies against oracle/_ref and tests/golden/).  Citations
 * are relative to /root/reference/.
 *
 * Return codes: 0 ok, 2 configuration error (the reference's ConfigError).
 */
#ifndef AFFMAE_ORACLE_H
#define AFFMAE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/geometry.cpp:15-30 */
uint64_t orc_hilbert_index(uint32_t n, uint32_t x, uint32_t y);
/* proj/src/geometry.cpp:57-106 (min_gap + sfc_order) */
int orc_sfc_order(const float* coords, int64_t n, int64_t* perm);
/* proj/src/geometry.cpp:108-131; returns the cluster count C (or -2) */
int64_t orc_balanced_clusters(const float* coords, int64_t n, int64_t size, int32_t* cluster_of,
                              int64_t* members, int64_t* member_off);
/* proj/src/geometry.cpp:133-186; nbr_cl [C, groups_eff]; idx/valid [n, width] */
int orc_cluster_neighborhood(const float* coords, int64_t n, int64_t c, const int64_t* members,
                             const int64_t* member_off, int64_t groups, int64_t* nbr_cl,
                             int64_t* idx, uint8_t* valid, int64_t width);
/* proj/src/geometry.cpp:188-216 */
int orc_knn(const float* queries, int64_t nq, const float* keys, int64_t nk, int64_t k,
            int64_t* idx, uint8_t* valid);

/* proj/src/attention.cpp:33-42 */
double orc_bias_eval(const float* w1, const float* b1, const float* w2, const float* b2,
                     int hidden, double patch, int head, double dx, double dy);
/* streaming_kernel<float> (proj/src/attention.cpp:119-185), b32 tensors */
int orc_attn_fwd_f32(int64_t n, int64_t m, int heads, int d, int hidden, double patch,
                     const float* q, const float* k, const float* v, const float* bk,
                     const float* bv, const float* coords, const int64_t* idx,
                     const uint8_t* valid, const float* w1, const float* b1, const float* w2,
                     const float* b2, const float* blank, float* out);
/* nbhd_attn_backward (proj/src/attention.cpp:241-358).  Inputs are the
 * tensor values as doubles; prec 32 reproduces the b32 gradient tensors
 * (every += rounds to binary32), prec 64 keeps binary64. */
int orc_attn_bwd(int64_t n, int64_t m, int heads, int d, int hidden, double patch, int prec,
                 const double* q, const double* k, const double* v, const double* bk,
                 const double* bv, const float* coords, const int64_t* idx,
                 const uint8_t* valid, const double* w1, const double* b1, const double* w2,
                 const double* b2, const double* blank, const double* dout, double* dq,
                 double* dk, double* dv, double* dbk, double* dbv, double* dw1, double* db1,
                 double* dw2, double* db2, double* dblank);

/* proj/src/merging.cpp:50-54 (-2 on bad d_s) */
int64_t orc_retained_count(int64_t n, double d_s);
/* proj/src/merging.cpp:56-69; returns the kept count */
int64_t orc_select_retained(const double* scores, int64_t n, double d_s, int64_t* out);
/* proj/src/merging.cpp:71-116 */
int orc_merge_plan(const float* coords, int64_t n, const int64_t* retained, int64_t r, int k_m,
                   int64_t* dropped, int64_t* target, int64_t* pool_idx, double* pool_dist,
                   int32_t* pool_cnt);
/* pool_forward (proj/src/merging.cpp:121-149) */
int orc_merge_pool_fwd(int64_t n, int64_t dim, int64_t r, int k_m, int prec,
                       const int64_t* retained, const int64_t* pool_idx, const double* pool_dist,
                       const int32_t* pool_cnt, const double* feats, const double* scores,
                       double p, double* out);
/* MergePoolOp::backward (proj/src/merging.cpp:169-219); accumulates (+=) */
int orc_merge_pool_bwd(int64_t n, int64_t dim, int64_t r, int k_m, int prec,
                       const int64_t* retained, const int64_t* pool_idx, const double* pool_dist,
                       const int32_t* pool_cnt, const double* feats, const double* scores,
                       double p, const double* dout, double* dfeats, double* dscores, double* dp);

/* make_interp_op forward / backward (interpolation.cpp:192-251) */
int orc_interp_fwd(int64_t nq, int64_t dim, int64_t k, int prec, const double* queries, const float* key_coords,
                   const double* feats, const int64_t* idx, const uint8_t* valid, double p, double eps,
                   double* out);
int orc_interp_bwd(int64_t nq, int64_t dim, int64_t k, const double* queries, const float* key_coords,
                   const double* feats, const int64_t* idx, const uint8_t* valid, double p, double eps,
                   const double* dout, double* dfeats, double* dp, double* dq);

/* AdamW::lr_at / AdamW::step (pipeline.cpp:643-680) */
double orc_adamw_lr(double lr, int64_t warmup, int64_t total, int64_t step);
int orc_adamw_step(double lr, int64_t warmup, double wd, double beta1, double beta2, int64_t total, int64_t step,
                   int64_t n_params, const int64_t* rows, const int64_t* cols, const double* grad, double* value,
                   double* m, double* v);

#ifdef __cplusplus
}
#endif
#endif
