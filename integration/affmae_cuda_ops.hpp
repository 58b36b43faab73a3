// affmae_cuda_ops.hpp -- reference-side adapters for libaffmae_b200.so.
//
// This is the binding a maintainer adds to the REFERENCE tree (it includes the
// reference's own headers): every factory/free function keeps the reference's
// signature and CustomOp semantics (include/affmae/tape.hpp:29-38 -- backward
// accumulates into non-null in_grads), but runs on the B200 through the C ABI
// declared in include/affmae_b200.h.  Host Tensors are copied to the device per
// call (bf16 activations, fp32 parameters), exactly the "host buffers" path.
// Status codes map back onto the reference taxonomy (ConfigError /
// NumericError, include/affmae/errors.hpp:8-15).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "affmae/attention.hpp"
#include "affmae/geometry.hpp"
#include "affmae/interpolation.hpp"
#include "affmae/masking.hpp"
#include "affmae/merging.hpp"
#include "affmae/tape.hpp"

namespace affmae::cuda {

// balanced_clusters / cluster_neighborhood (include/affmae/geometry.hpp:61-68)
ClusterAssignment balanced_clusters(const PointSet& points, int64_t size);
NeighborIndex cluster_neighborhood_from_coords(const PointSet& points, int64_t size, int64_t groups);
// cluster_neighborhood with the reference's signature (include/affmae/geometry.hpp:67)
NeighborIndex cluster_neighborhood(const ClusterAssignment& assign, const PointSet& points, int64_t groups);
// sfc_order / knn (include/affmae/geometry.hpp:59,72)
std::vector<int64_t> sfc_order(const PointSet& points);
NeighborIndex knn(const Tensor& queries, const PointSet& keys, int64_t k);

// Cluster attention as a tape op (make_attn_op, include/affmae/attention.hpp:84-86).
// The cluster structure (size, groups) is what Model::encode passes to
// balanced_clusters/cluster_neighborhood right before building the op
// (proj/src/pipeline.cpp:442-444); the device index is rebuilt from `coords`.
std::shared_ptr<CustomOp> make_cluster_attn_op(Tensor coords, int64_t cluster, int64_t groups,
                                               int heads, int head_dim, int bias_hidden,
                                               double patch);

// make_attn_op with the reference's exact signature (include/affmae/attention.hpp:84-86), a
// drop-in for Model::attn_layer (src/pipeline.cpp:379-386).  A NeighborIndex that is a
// cluster_neighborhood index of `coords` (detected: rebuilt on the device for the (size,
// groups) its width allows and compared entry for entry) runs on the cluster kernels with
// the frozen plan; any other index of width <= 31 (the decoder's one_to_one / knn rows,
// src/pipeline.cpp:515-525) on the general-row kernels; anything else is a ConfigError.
std::shared_ptr<CustomOp> make_attn_op(Tensor coords, NeighborIndex nbr, int heads, int head_dim,
                                       int bias_hidden, double patch, bool streaming = true,
                                       bool half_io = false);
// the two device paths, explicitly
std::shared_ptr<CustomOp> make_general_attn_op(Tensor coords, NeighborIndex nbr, int heads, int head_dim,
                                               int bias_hidden, double patch);

// Device-generated inputs: mask_from_field(perlin_field(hp, wp, kPerlinOctaves, kPerlinBaseFreq,
// kPerlinPersistence, seed), ratio) (include/affmae/masking.hpp:31-40; bit-exact) and
// synth_image (include/affmae/pipeline.hpp:30; within 1e-12).
MaskSpec perlin_mask(int64_t hp, int64_t wp, double ratio, uint64_t seed);
Tensor synth_image(int64_t size, uint64_t seed);

// select_retained / merge_plan / make_merge_pool_op (include/affmae/merging.hpp:32-68)
std::vector<int64_t> select_retained(const Tensor& scores, double d_s);
MergePlan merge_plan(const PointSet& ps, std::span<const int64_t> retained, int k_m);
std::shared_ptr<CustomOp> make_merge_pool_op(MergePlan plan);

// Softmax interpolation tape op (make_interp_op, include/affmae/interpolation.hpp:60):
// inputs {feats NxD, p 1x1, queries Qx2}; neighbour rows frozen at construction
// (width <= 32), gradients to feats, p and the query coordinates.
std::shared_ptr<CustomOp> make_interp_op(Tensor key_coords, NeighborIndex nbrs, double eps = kInterpEps);

}  // namespace affmae::cuda
