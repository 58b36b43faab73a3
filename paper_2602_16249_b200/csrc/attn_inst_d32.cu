// Explicit instantiations of the attention kernels for head_dim 32
// (split across translation units so the build parallelises).
#include "attn_kernels.cuh"

namespace affmae_b200 {
AFFMAE_INSTANTIATE_ATTN_QK(32, 16)
AFFMAE_INSTANTIATE_ATTN_QK(32, 32)
AFFMAE_INSTANTIATE_ATTN_QK(32, 48)
AFFMAE_INSTANTIATE_ATTN_QK(32, 64)
AFFMAE_INSTANTIATE_ATTN_KV(32)
}  // namespace affmae_b200
