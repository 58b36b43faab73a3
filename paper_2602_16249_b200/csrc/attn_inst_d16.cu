// Explicit instantiations of the attention kernels for head_dim 16
// (split across translation units so the build parallelises).
#include "attn_kernels.cuh"

namespace affmae_b200 {
AFFMAE_INSTANTIATE_ATTN(16, 4, 1)
AFFMAE_INSTANTIATE_ATTN(16, 4, 2)
AFFMAE_INSTANTIATE_ATTN(16, 4, 4)
AFFMAE_INSTANTIATE_ATTN(16, 7, 1)
AFFMAE_INSTANTIATE_ATTN(16, 7, 2)
AFFMAE_INSTANTIATE_ATTN(16, 7, 4)
}  // namespace affmae_b200
