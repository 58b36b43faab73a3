// Test shim: runs the REFERENCE's own Tape (proj/src/tape.cpp) with either the
// reference CPU ops or the B200 ops from affmae_cuda_ops.hpp plugged in, so a
// GPU test can check the drop-in at the CustomOp boundary.
#include <cstring>
#include <exception>
#include <string>

#include "affmae/attention.hpp"
#include "affmae/errors.hpp"
#include "affmae/geometry.hpp"
#include "affmae/masking.hpp"
#include "affmae/merging.hpp"
#include "affmae/pipeline.hpp"
#include "affmae/tape.hpp"
#include "affmae_cuda_ops.hpp"

using namespace affmae;

namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
Tensor from(const double* p, std::vector<int64_t> dims) {
    Tensor t = Tensor::zeros(std::move(dims), Precision::b32);
    for (int64_t i = 0; i < t.numel(); ++i) t.set(i, p[i]);
    return t;
}
void to(const Tensor& t, double* o) {
    for (int64_t i = 0; i < t.numel(); ++i) o[i] = t.get(i);
}
PointSet pts(const float* c, int64_t n) {
    PointSet ps;
    ps.coords = Tensor::zeros({n, 2}, Precision::b32);
    for (int64_t i = 0; i < 2 * n; ++i) ps.coords.set(i, c[i]);
    ps.feats = Tensor::zeros({n, 0}, Precision::b32);
    return ps;
}
}  // namespace

extern "C" {

const char* integ_last_error() { return g_err.c_str(); }

// Geometry through the adapters vs the reference: returns the number of mismatches.
int integ_geometry(const float* coords, int64_t n, int64_t size, int64_t groups, int64_t* mismatches) {
    return guarded([&] {
        PointSet ps = pts(coords, n);
        int64_t bad = 0;
        auto o1 = sfc_order(ps), o2 = cuda::sfc_order(ps);
        bad += o1 != o2;
        ClusterAssignment a1 = balanced_clusters(ps, size), a2 = cuda::balanced_clusters(ps, size);
        bad += a1.cluster_of != a2.cluster_of;
        bad += a1.members != a2.members;
        NeighborIndex n1 = cluster_neighborhood(a1, ps, groups);
        NeighborIndex n2 = cuda::cluster_neighborhood_from_coords(ps, size, groups);
        bad += n1.width != n2.width || n1.valid != n2.valid;
        for (size_t i = 0; i < n1.idx.size() && i < n2.idx.size(); ++i) bad += n1.valid[i] && n1.idx[i] != n2.idx[i];
        NeighborIndex k1 = knn(ps.coords, ps, 8), k2 = cuda::knn(ps.coords, ps, 8);
        bad += k1.idx != k2.idx || k1.valid != k2.valid;
        *mismatches = bad;
    });
}

// One attention layer on the reference Tape: out = op(q, k, v, ...), loss = sum(out * w),
// backward.  use_cuda selects the B200 op; otherwise the reference's make_attn_op with
// cluster_neighborhood.  Outputs: out [n, h*d] and the 10 input gradients.
int integ_attn_tape(int use_cuda, int64_t n, int heads, int d, int hidden, double patch, int64_t cluster,
                    int64_t groups, const float* coords, const double* const* ins, const double* w,
                    double* out, double* const* grads) {
    return guarded([&] {
        const int64_t hd = int64_t(heads) * d;
        std::vector<std::vector<int64_t>> dims = {{n, hd}, {n, hd}, {n, hd}, {heads, d}, {heads, d},
                                                  {heads, 2 * hidden}, {heads, hidden}, {heads, hidden},
                                                  {heads, 1}, {heads, 1}};
        Tape t(Precision::b32);
        std::vector<int> ids;
        for (int i = 0; i < 10; ++i) ids.push_back(t.leaf(from(ins[i], dims[size_t(i)])));
        PointSet ps = pts(coords, n);
        std::shared_ptr<CustomOp> op;
        if (use_cuda == 2) {  // the reference's exact call, namespace-qualified (drop-in detection)
            ClusterAssignment a = cuda::balanced_clusters(ps, cluster);
            op = cuda::make_attn_op(ps.coords, cuda::cluster_neighborhood(a, ps, groups), heads, d, hidden, patch);
        } else if (use_cuda) {
            op = cuda::make_cluster_attn_op(ps.coords, cluster, groups, heads, d, hidden, patch);
        } else {
            ClusterAssignment a = balanced_clusters(ps, cluster);
            op = make_attn_op(ps.coords, cluster_neighborhood(a, ps, groups), heads, d, hidden, patch);
        }
        int o = t.custom(op, ids);
        int loss = t.reduce_sum(t.mul(o, t.input(from(w, {n, hd}))));
        t.backward(loss);
        to(t.value(o), out);
        for (int i = 0; i < 10; ++i) to(t.grad(ids[size_t(i)]), grads[i]);
    });
}

// Merge on the reference Tape: retained = select_retained(scores), plan = merge_plan,
// pooled = pool(feats, scores, p), loss = sum(pooled * w), backward.
int integ_merge_tape(int use_cuda, int64_t n, int64_t dim, double d_s, int k_m, const float* coords,
                     const double* feats, const double* scores, double p, const double* w, int64_t* retained,
                     int64_t* n_ret, int64_t* pool_idx, double* pooled, double* dfeats, double* dscores,
                     double* dp) {
    return guarded([&] {
        PointSet ps = pts(coords, n);
        Tensor sc = from(scores, {n, 1});
        std::vector<int64_t> r = use_cuda ? cuda::select_retained(sc, d_s) : select_retained(sc, d_s);
        MergePlan plan = use_cuda ? cuda::merge_plan(ps, r, k_m) : merge_plan(ps, r, k_m);
        *n_ret = int64_t(r.size());
        for (size_t i = 0; i < r.size(); ++i) retained[i] = r[i];
        for (size_t i = 0; i < r.size(); ++i)
            for (int t2 = 0; t2 < k_m; ++t2)
                pool_idx[i * size_t(k_m) + size_t(t2)] = size_t(t2) < plan.pool[i].size() ? plan.pool[i][size_t(t2)] : -1;
        Tape t(Precision::b32);
        int f = t.leaf(from(feats, {n, dim})), s = t.leaf(sc), pp = t.leaf(Tensor::full({1, 1}, p, Precision::b32));
        auto op = use_cuda ? cuda::make_merge_pool_op(plan) : make_merge_pool_op(plan);
        int o = t.custom(op, {f, s, pp});
        int loss = t.reduce_sum(t.mul(o, t.input(from(w, {int64_t(r.size()), 2 * dim}))));
        t.backward(loss);
        to(t.value(o), pooled);
        to(t.grad(f), dfeats);
        to(t.grad(s), dscores);
        *dp = t.grad(pp).get(0);
    });
}

// Decoder-style interpolation on the reference Tape: nbrs = knn(queries, keys, k),
// out = interp(feats, p, queries), loss = sum(out * w), backward.
int integ_interp_tape(int use_cuda, int64_t nk, int64_t nq, int64_t dim, int64_t k, const float* keys,
                      const double* queries, const double* feats, double p, const double* w, double* out,
                      double* dfeats, double* dp, double* dq) {
    return guarded([&] {
        PointSet ks = pts(keys, nk);
        Tensor qt = from(queries, {nq, 2});
        NeighborIndex nb = use_cuda ? cuda::knn(qt, ks, k) : knn(qt, ks, k);
        Tape t(Precision::b32);
        int f = t.leaf(from(feats, {nk, dim})), pp = t.leaf(Tensor::full({1, 1}, p, Precision::b32)), q = t.leaf(qt);
        auto op = use_cuda ? cuda::make_interp_op(ks.coords, nb) : make_interp_op(ks.coords, nb);
        int o = t.custom(op, {f, pp, q});
        int loss = t.reduce_sum(t.mul(o, t.input(from(w, {nq, dim}))));
        t.backward(loss);
        to(t.value(o), out);
        to(t.grad(f), dfeats);
        *dp = t.grad(pp).get(0);
        to(t.grad(q), dq);
    });
}

// Decoder self attention on the reference Tape: nbr = knn(coords, coords, k) (the
// decoder's self_nbr, src/pipeline.cpp:493), out = attn(q, k, v, ...), loss = sum(out * w).
int integ_gattn_tape(int use_cuda, int64_t n, int heads, int d, int hidden, double patch, int64_t k,
                     const float* coords, const double* const* ins, const double* w, double* out,
                     double* const* grads) {
    return guarded([&] {
        const int64_t hd = int64_t(heads) * d;
        std::vector<std::vector<int64_t>> dims = {{n, hd}, {n, hd}, {n, hd}, {heads, d}, {heads, d},
                                                  {heads, 2 * hidden}, {heads, hidden}, {heads, hidden},
                                                  {heads, 1}, {heads, 1}};
        Tape t(Precision::b32);
        std::vector<int> ids;
        for (int i = 0; i < 10; ++i) ids.push_back(t.leaf(from(ins[i], dims[size_t(i)])));
        PointSet ps = pts(coords, n);
        NeighborIndex nb = use_cuda ? cuda::knn(ps.coords, ps, k) : knn(ps.coords, ps, k);
        auto op = use_cuda ? cuda::make_attn_op(ps.coords, nb, heads, d, hidden, patch)
                           : make_attn_op(ps.coords, nb, heads, d, hidden, patch);
        int o = t.custom(op, ids);
        int loss = t.reduce_sum(t.mul(o, t.input(from(w, {n, hd}))));
        t.backward(loss);
        to(t.value(o), out);
        for (int i = 0; i < 10; ++i) to(t.grad(ids[size_t(i)]), grads[i]);
    });
}

// Perlin mask and synthetic image through either side's public functions.
int integ_inputs(int use_cuda, int64_t grid, double ratio, uint64_t seed, uint8_t* mask, int64_t img_size,
                 double* img) {
    return guarded([&] {
        MaskSpec m = use_cuda ? cuda::perlin_mask(grid, grid, ratio, seed)
                              : mask_from_field(perlin_field(grid, grid, kPerlinOctaves, kPerlinBaseFreq,
                                                             kPerlinPersistence, seed),
                                                ratio);
        for (size_t i = 0; i < m.masked.size(); ++i) mask[i] = m.masked[i];
        Tensor t = use_cuda ? cuda::synth_image(img_size, seed) : synth_image(img_size, seed);
        to(t, img);
    });
}

}  // extern "C"
