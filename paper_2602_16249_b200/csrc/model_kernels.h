// Row / elementwise kernels of the training step (model_kernels.cu); host launchers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace affmae_b200 {
namespace mk {

using bf16 = __nv_bfloat16;

// LayerNorm over fp32 rows (optionally x + add first, the sum stored to xo / xo_bf), y bf16,
// stats {mean, rstd}; widths 64 * {1,2,3,4,6,8,12,16}
int ln_fwd(const float* x, const bf16* add, float* xo, bf16* xo_bf, const float* g, const float* b, int64_t rows,
           int64_t C, bf16* y, float2* stats, cudaStream_t st);
int ln_fwd_bf(const bf16* x, float* xo, const float* g, const float* b, int64_t rows, int64_t C, bf16* y,
              float2* stats, cudaStream_t st);
// VJP fused with the residual-gradient sum: dres_out = dres_in + dx (either may be null),
// optional bf16 copy; dgamma / dbeta ACCUMULATED (+=) through `part` (ln_bwd_part_floats)
int ln_bwd(const float* dy, const float* x, const float2* stats, const float* g, int64_t rows, int64_t C,
           const float* dres_in, float* dres_out, bf16* dres_bf, float* dgamma, float* dbeta, float* part,
           cudaStream_t st);
int ln_bwd_bf(const float* dy, const bf16* x, const float2* stats, const float* g, int64_t rows, int64_t C,
              const float* dres_in, float* dres_out, bf16* dres_bf, float* dgamma, float* dbeta, float* part,
              cudaStream_t st);
size_t ln_bwd_part_floats(int64_t rows, int64_t C);

// positional MLP first layer: H = GELU((coords * inv_image) W1^T + b1) [rows, 16] bf16
int pos_hidden_fwd(const float* coords, int64_t rows, float inv_image, const float* w1, const float* b1, bf16* h,
                   cudaStream_t st);
// dW1 / db1 += from dH [rows, 16] fp32; part >= pos_part_floats(rows)
int pos_hidden_bwd(const float* coords, int64_t rows, float inv_image, const float* w1, const float* b1,
                   const float* dh, float* dw1, float* db1, float* part, cudaStream_t st);
unsigned pos_bwd_blocks(int64_t rows);
inline size_t pos_part_floats(int64_t rows) { return size_t(pos_bwd_blocks(rows)) * 48; }

// merge scorer output unit: scores = sigmoid(hid . w2 + b2); backward writes dhid (bf16)
// and accumulates dw2 / db2
int scorer_out_fwd(const bf16* hid, int64_t rows, const float* w2, const float* b2, float* scores, cudaStream_t st);
int scorer_out_bwd(const bf16* hid, const float* scores, const float* dscores, int64_t rows, const float* w2,
                   bf16* dhid, float* dw2, float* db2, float* part, cudaStream_t st);

// decoder offset head (linear dd -> 2 + NormClampOp) and its VJP (dfq += in place)
int offset_fwd(const float* fq, int64_t rows, int64_t C, const float* w, const float* b, double limit,
               const float* refs, float* pre, float* qpos, cudaStream_t st);
int offset_bwd(const float* fq, int64_t rows, int64_t C, const float* w, double limit, const float* pre,
               const float* dqpos, float* dfq, float* dw, float* db, float* part, cudaStream_t st);
unsigned offset_bwd_blocks(int64_t rows);
inline size_t offset_part_floats(int64_t rows, int64_t C) { return size_t(offset_bwd_blocks(rows)) * (2 * C + 2); }

// cells with mask byte == want, ascending, n per image: global rows and pixel centres
int cell_rows(const uint8_t* masked, int64_t batch, int64_t gh, int64_t gw, int want, int64_t n, double patch,
              int32_t* rows, float* coords, cudaStream_t st);
int gather_rows_bf16(const float* src, const int32_t* rows, int64_t n, int64_t p2, bf16* out, cudaStream_t st);
int gather_coords(const float* coords, const int32_t* ret, int64_t batch, int64_t n, int64_t r, float* out,
                  cudaStream_t st);

int add_f32_bf16(const float* a, int a_row, const bf16* b, int64_t rows, int64_t cols, float* out, bf16* out_bf,
                 cudaStream_t st);
int cast_bf16(const float* x, int64_t n, bf16* y, cudaStream_t st);
int cast_bf16_2d(const float* x, int64_t rows, int64_t cols, bf16* y, int64_t ldy, cudaStream_t st);
int gelu_fwd(const bf16* pre, int64_t n, bf16* y, cudaStream_t st);
int colsum_f32(const float* x, int64_t rows, int64_t cols, float* out, float* part, cudaStream_t st);
size_t colsum_part_floats(int64_t cols);
int shadow_cast(const float* p, int64_t n, bf16* pb, cudaStream_t st);

}  // namespace mk
}  // namespace affmae_b200
