// Definitions behind redirect_b200.hpp: the renamed declarations the reference's pipeline.cpp
// now calls, forwarding to the B200 adapters with the reference's signatures unchanged.
#include "affmae_cuda_ops.hpp"

namespace affmae {

ClusterAssignment b200_balanced_clusters(const PointSet& points, int64_t size) {
    return cuda::balanced_clusters(points, size);
}
NeighborIndex b200_cluster_neighborhood(const ClusterAssignment& assign, const PointSet& points, int64_t groups) {
    return cuda::cluster_neighborhood(assign, points, groups);
}
std::shared_ptr<CustomOp> b200_make_attn_op(Tensor coords, NeighborIndex nbr, int heads, int head_dim,
                                            int bias_hidden, double patch, bool streaming, bool half_io) {
    return cuda::make_attn_op(std::move(coords), std::move(nbr), heads, head_dim, bias_hidden, patch, streaming,
                              half_io);
}
std::vector<int64_t> b200_select_retained(const Tensor& scores, double d_s) {
    return cuda::select_retained(scores, d_s);
}
MergePlan b200_merge_plan(const PointSet& ps, std::span<const int64_t> retained, int k_m) {
    return cuda::merge_plan(ps, retained, k_m);
}
std::shared_ptr<CustomOp> b200_make_merge_pool_op(MergePlan plan) { return cuda::make_merge_pool_op(std::move(plan)); }
NeighborIndex b200_knn(const Tensor& queries, const PointSet& keys, int64_t k) { return cuda::knn(queries, keys, k); }
std::shared_ptr<CustomOp> b200_make_interp_op(Tensor key_coords, NeighborIndex nbrs, double eps) {
    return cuda::make_interp_op(std::move(key_coords), std::move(nbrs), eps);
}

}  // namespace affmae
