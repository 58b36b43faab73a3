// Explicit instantiations of the attention kernels for head_dim 16
// (split across translation units so the build parallelises).
#include "attn_kernels.cuh"

namespace affmae_b200 {
AFFMAE_INSTANTIATE_ATTN_QK(16, 16)
AFFMAE_INSTANTIATE_ATTN_QK(16, 32)
AFFMAE_INSTANTIATE_ATTN_QK(16, 48)
AFFMAE_INSTANTIATE_ATTN_QK(16, 64)
AFFMAE_INSTANTIATE_ATTN_KV(16)
}  // namespace affmae_b200
