// Force-included (g++ -include) when the drop-in test compiles the reference's UNMODIFIED
// src/pipeline.cpp where it lies: the hot-path names Model::encode / decode / deep_sup call
// (src/pipeline.cpp:379-386, 442-457, 495-535, 572-576) resolve to the B200 adapters below --
// the effect of a maintainer qualifying those calls with `cuda::` (affmae_cuda_ops.hpp).
// Nothing else of the reference changes.
#pragma once
#define balanced_clusters b200_balanced_clusters
#define cluster_neighborhood b200_cluster_neighborhood
#define make_attn_op b200_make_attn_op
#define select_retained b200_select_retained
#define merge_plan b200_merge_plan
#define make_merge_pool_op b200_make_merge_pool_op
#define knn b200_knn
#define make_interp_op b200_make_interp_op
