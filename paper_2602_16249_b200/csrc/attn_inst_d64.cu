// Explicit instantiations of the attention kernels for head_dim 64
// (split across translation units so the build parallelises).
#include "attn_kernels.cuh"

namespace affmae_b200 {
AFFMAE_INSTANTIATE_ATTN_QK(64, 16)
AFFMAE_INSTANTIATE_ATTN_QK(64, 32)
AFFMAE_INSTANTIATE_ATTN_QK(64, 48)
AFFMAE_INSTANTIATE_ATTN_QK(64, 64)
AFFMAE_INSTANTIATE_ATTN_KV(64)
}  // namespace affmae_b200
