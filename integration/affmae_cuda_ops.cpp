// Reference-side adapters over the B200 C ABI (see affmae_cuda_ops.hpp).
#include "affmae_cuda_ops.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "affmae/errors.hpp"
#include "affmae_b200.h"

namespace affmae::cuda {
namespace {

void check(int rc, const char* what) {
    if (rc == AFFMAE_OK) return;
    std::string msg = std::string(what) + ": " + affmae_last_error();
    if (rc == AFFMAE_ECONFIG || rc == AFFMAE_EUNSUPPORTED) throw ConfigError(msg);
    if (rc == AFFMAE_ENUMERIC) throw NumericError(msg);
    throw std::runtime_error(msg);
}
void ccheck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// owning device buffer
struct Dev {
    void* p = nullptr;
    size_t n = 0;
    explicit Dev(size_t bytes) : n(bytes) { ccheck(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    template <class T> T* as() const { return static_cast<T*>(p); }
};

template <class T>
std::unique_ptr<Dev> upload(const std::vector<T>& h) {
    auto d = std::make_unique<Dev>(h.size() * sizeof(T));
    ccheck(cudaMemcpy(d->p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    return d;
}
template <class T>
std::vector<T> download(const Dev& d, size_t n) {
    std::vector<T> h(n);
    ccheck(cudaMemcpy(h.data(), d.p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    return h;
}
std::vector<float> f32(const Tensor& t) {
    std::vector<float> v(size_t(t.numel()));
    for (int64_t i = 0; i < t.numel(); ++i) v[size_t(i)] = float(t.get(i));
    return v;
}
std::vector<uint16_t> bf16(const Tensor& t) {
    std::vector<uint16_t> v(size_t(t.numel()));
    for (int64_t i = 0; i < t.numel(); ++i) {
        __nv_bfloat16 b = __float2bfloat16(float(t.get(i)));
        std::memcpy(&v[size_t(i)], &b, 2);
    }
    return v;
}
float bf16_to_float(uint16_t u) {
    uint32_t x = uint32_t(u) << 16;
    float f;
    std::memcpy(&f, &x, 4);
    return f;
}

// [rows, groups*w] -> bf16 [rows, groups*wp] (each group zero-padded to wp, times scale): head
// dims / feature widths the reference allows but the kernels are not compiled for (e.g. the
// toy() config's head_dim 12) run on the next compiled width with zero padding
std::vector<uint16_t> bf16_pad(const Tensor& t, int64_t groups, int64_t w, int64_t wp, float scale = 1.f) {
    const int64_t rows = t.numel() / (groups * w);
    std::vector<uint16_t> v(size_t(rows * groups * wp), 0);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t g = 0; g < groups; ++g)
            for (int64_t e = 0; e < w; ++e) {
                __nv_bfloat16 b = __float2bfloat16(float(t.get((r * groups + g) * w + e)) * scale);
                std::memcpy(&v[size_t((r * groups + g) * wp + e)], &b, 2);
            }
    return v;
}
// value of padded element (r, g, e) of a [rows, groups*wp] array
inline int64_t pad_at(int64_t r, int64_t g, int64_t e, int64_t groups, int64_t wp) { return (r * groups + g) * wp + e; }
int padded_head_dim(int d) {
    if (d <= 16) return 16;
    if (d <= 32) return 32;
    if (d <= 64) return 64;
    throw ConfigError("attention op: head_dim > 64 not compiled");
}

struct DeviceIndex {
    affmae_cluster_geom g{};
    std::unique_ptr<Dev> perm, cof, nbr, roff, rcl;
    affmae_cluster_index idx{};
};

DeviceIndex build_index(const Dev& coords, int64_t n, int64_t size, int64_t groups) {
    DeviceIndex d;
    d.g.batch = 1;
    d.g.tokens = n;
    d.g.cluster = size;
    d.g.groups = groups;
    check(affmae_cluster_geometry(&d.g), "cluster_geometry");
    d.perm = std::make_unique<Dev>(n * 4);
    d.cof = std::make_unique<Dev>(n * 4);
    d.nbr = std::make_unique<Dev>(d.g.n_clusters * d.g.groups_eff * 4);
    d.roff = std::make_unique<Dev>((d.g.n_clusters + 1) * 4);
    d.rcl = std::make_unique<Dev>(d.g.n_clusters * d.g.groups_eff * 4);
    d.idx = {d.perm->as<int32_t>(), d.cof->as<int32_t>(), d.nbr->as<int32_t>(), d.roff->as<int32_t>(),
             d.rcl->as<int32_t>()};
    Dev ws(affmae_cluster_index_workspace(&d.g));
    check(affmae_cluster_index_build(&d.g, coords.as<float>(), &d.idx, ws.p, ws.n, nullptr), "cluster_index_build");
    return d;
}

}  // namespace

ClusterAssignment balanced_clusters(const PointSet& points, int64_t size) {
    const int64_t n = points.count();
    if (size < 1) throw ConfigError("balanced_clusters: size must be >= 1");
    auto c = upload(f32(points.coords));
    DeviceIndex d = build_index(*c, n, size, 1);
    ccheck(cudaDeviceSynchronize(), "sync");
    auto perm = download<int32_t>(*d.perm, size_t(n));
    ClusterAssignment a;
    a.target = std::min(size, n);
    a.cluster_of = download<int32_t>(*d.cof, size_t(n));
    a.members.resize(size_t(d.g.n_clusters));
    const int64_t base = n / d.g.n_clusters, rem = n % d.g.n_clusters;
    int64_t pos = 0;
    for (int64_t k = 0; k < d.g.n_clusters; ++k)
        for (int64_t j = 0; j < base + (k < rem ? 1 : 0); ++j) a.members[size_t(k)].push_back(perm[size_t(pos++)]);
    return a;
}

NeighborIndex cluster_neighborhood_from_coords(const PointSet& points, int64_t size, int64_t groups) {
    const int64_t n = points.count();
    auto c = upload(f32(points.coords));
    DeviceIndex d = build_index(*c, n, size, groups);
    const int64_t m = d.g.width;
    Dev idx(n * m * 4), valid(n * m);
    check(affmae_neighbor_expand(&d.g, d.perm->as<int32_t>(), d.nbr->as<int32_t>(), idx.as<int32_t>(),
                                 valid.as<uint8_t>(), nullptr), "neighbor_expand");
    ccheck(cudaDeviceSynchronize(), "sync");
    NeighborIndex nb;
    nb.width = m;
    auto hi = download<int32_t>(idx, size_t(n * m));
    auto hv = download<uint8_t>(valid, size_t(n * m));
    nb.idx.assign(hi.begin(), hi.end());
    nb.valid.assign(hv.begin(), hv.end());
    return nb;
}

NeighborIndex cluster_neighborhood(const ClusterAssignment& assign, const PointSet& points, int64_t groups) {
    // the device rebuilds the assignment from the coordinates (balanced_clusters(points,
    // assign.target)); an assignment from anywhere else is a ConfigError, not a silent mismatch
    if (groups < 1) throw ConfigError("cluster_neighborhood: groups must be >= 1");
    ClusterAssignment mine = cuda::balanced_clusters(points, assign.target);
    if (mine.cluster_of != assign.cluster_of)
        throw ConfigError("cuda::cluster_neighborhood: assignment is not balanced_clusters(points, target)");
    return cluster_neighborhood_from_coords(points, assign.target, groups);
}

std::vector<int64_t> sfc_order(const PointSet& points) {
    const int64_t n = points.count();
    if (n < 1) throw ConfigError("sfc_order: empty point set");
    auto c = upload(f32(points.coords));
    Dev perm(n * 4), ws(affmae_sfc_order_workspace(1, n));
    check(affmae_sfc_order(c->as<float>(), 1, n, perm.as<int32_t>(), ws.p, ws.n, nullptr), "sfc_order");
    auto h = download<int32_t>(perm, size_t(n));
    return std::vector<int64_t>(h.begin(), h.end());
}

NeighborIndex knn(const Tensor& queries, const PointSet& keys, int64_t k) {
    const int64_t nq = queries.dim(0), nk = keys.count();
    auto q = upload(f32(queries));
    auto kk = upload(f32(keys.coords));
    Dev idx(std::max<int64_t>(nq * k, 1) * 4), valid(std::max<int64_t>(nq * k, 1));
    check(affmae_knn(q->as<float>(), kk->as<float>(), 1, nq, nk, k, idx.as<int32_t>(), valid.as<uint8_t>(), nullptr), "knn");
    NeighborIndex nb;
    nb.width = k;
    auto hi = download<int32_t>(idx, size_t(nq * k));
    auto hv = download<uint8_t>(valid, size_t(nq * k));
    nb.idx.assign(hi.begin(), hi.end());
    nb.valid.assign(hv.begin(), hv.end());
    return nb;
}

namespace {

// Tape op: inputs {q, k, v, blank_k, blank_v, w1, b1, w2, b2, blank}
// (src/attention.cpp:374-444 ordering).  Like the reference's AttnOp, the op's
// geometry is frozen: the device coordinates, the cluster index and the
// attention plan (affmae_attn_plan_build) are built once, on first use, and
// reused by every forward and backward of the op.
struct ClusterAttnOp final : CustomOp {
    Tensor coords;
    int64_t cluster, groups;
    int heads, head_dim, hidden;
    double patch;

    struct Geometry {
        std::unique_ptr<Dev> coords;
        DeviceIndex d;
        std::unique_ptr<Dev> plan_buf;
        affmae_attn_plan plan{};
    };
    std::shared_ptr<Geometry> geo;

    std::string name() const override { return "cluster_attention_b200"; }

    // the device head dim (head_dim zero-padded to a compiled width); q carries the scale
    // sqrt(dp / head_dim) so the kernel's 1/sqrt(dp) gives the reference's 1/sqrt(head_dim)
    int dp() const { return padded_head_dim(head_dim); }
    float qscale() const { return float(std::sqrt(double(dp()) / double(head_dim))); }
    affmae_attn_desc desc() const { return {heads, dp(), hidden, patch}; }

    Geometry& geometry(int64_t n) {
        if (!geo) {
            auto g = std::make_shared<Geometry>();
            g->coords = upload(f32(coords));
            g->d = build_index(*g->coords, n, cluster, groups);
            affmae_attn_desc a = desc();
            g->plan_buf = std::make_unique<Dev>(affmae_attn_plan_workspace(&g->d.g, 1));
            g->plan.buf = g->plan_buf->p;
            g->plan.bytes = g->plan_buf->n;
            check(affmae_attn_plan_build(&g->d.g, &a, g->coords->as<float>(), &g->d.idx, 1, &g->plan, nullptr),
                  "attn_plan_build");
            geo = g;
        }
        return *geo;
    }

    // uploads the 10 inputs; `t` owns the device copies
    affmae_attn_inputs inputs(const std::vector<const Tensor*>& in, Geometry& G, std::unique_ptr<Dev> (&t)[10]) {
        t[0] = upload(bf16_pad(*in[0], heads, head_dim, dp(), qscale()));
        for (int i = 1; i < 3; ++i) t[i] = upload(bf16_pad(*in[size_t(i)], heads, head_dim, dp()));
        for (int i = 3; i < 5; ++i) t[i] = upload(bf16_pad(*in[size_t(i)], 1, head_dim, dp()));
        for (int i = 5; i < 10; ++i) t[i] = upload(f32(*in[size_t(i)]));
        return {t[0]->as<affmae_bf16>(), t[1]->as<affmae_bf16>(), t[2]->as<affmae_bf16>(),
                t[3]->as<affmae_bf16>(), t[4]->as<affmae_bf16>(), G.coords->as<float>(),
                t[5]->as<float>(), t[6]->as<float>(), t[7]->as<float>(), t[8]->as<float>(),
                t[9]->as<float>()};
    }

    void run_forward(Geometry& G, const affmae_attn_inputs& ai, Dev& out, Dev& lse) {
        affmae_attn_desc a = desc();
        Dev ws(affmae_attn_fwd_planned_workspace(&G.d.g, &a));
        check(affmae_attn_fwd_planned(&G.d.g, &a, &ai, &G.plan, out.as<affmae_bf16>(), lse.as<float>(), ws.p, ws.n,
                                      nullptr),
              "attn_fwd");
    }

    // Activations of the last forward, kept on the device for the backward (the Tape calls
    // backward with the same inputs, include/affmae/tape.hpp:32-38): the inputs' device copies,
    // O and LSE -- the backward neither re-uploads nor recomputes the forward.
    struct Saved {
        std::unique_ptr<Dev> t[10], out, lse;
        affmae_attn_inputs ai{};
        const Tensor* src[10] = {};
    };
    std::unique_ptr<Saved> saved;

    bool same_inputs(const std::vector<const Tensor*>& in) const {
        if (!saved) return false;
        for (int i = 0; i < 10; ++i)
            if (saved->src[i] != in[size_t(i)]) return false;
        return true;
    }

    Tensor forward(const std::vector<const Tensor*>& in) override {
        if (in.size() != 10) throw ConfigError("attention op: want 10 inputs");
        const int64_t n = in[0]->rows(), hd = int64_t(heads) * head_dim, hdp = int64_t(heads) * dp();
        Geometry& G = geometry(n);
        auto sv = std::make_unique<Saved>();
        sv->ai = inputs(in, G, sv->t);
        for (int i = 0; i < 10; ++i) sv->src[i] = in[size_t(i)];
        sv->out = std::make_unique<Dev>(n * hdp * 2);
        sv->lse = std::make_unique<Dev>(n * heads * 4);
        run_forward(G, sv->ai, *sv->out, *sv->lse);
        auto h = download<uint16_t>(*sv->out, size_t(n * hdp));
        Tensor o = Tensor::zeros({n, hd}, in[0]->precision());
        for (int64_t r = 0; r < n; ++r)
            for (int g = 0; g < heads; ++g)
                for (int e = 0; e < head_dim; ++e)
                    o.set((r * heads + g) * head_dim + e, bf16_to_float(h[size_t(pad_at(r, g, e, heads, dp()))]));
        saved = std::move(sv);
        return o;
    }

    void backward(const Tensor& out_grad, const std::vector<const Tensor*>& in,
                  const std::vector<Tensor*>& in_grads) override {
        const int64_t n = in[0]->rows(), hd = int64_t(heads) * dp();
        Geometry& G = geometry(n);
        affmae_attn_desc a = desc();
        if (!same_inputs(in)) {  // not the tensors of the last forward: rebuild the saved state
            auto sv = std::make_unique<Saved>();
            sv->ai = inputs(in, G, sv->t);
            for (int i = 0; i < 10; ++i) sv->src[i] = in[size_t(i)];
            sv->out = std::make_unique<Dev>(n * hd * 2);
            sv->lse = std::make_unique<Dev>(n * heads * 4);
            run_forward(G, sv->ai, *sv->out, *sv->lse);
            saved = std::move(sv);
        }
        Saved& S = *saved;
        auto dout = upload(bf16_pad(out_grad, heads, head_dim, dp()));
        Dev dq(n * hd * 2), dk(n * hd * 2), dv(n * hd * 2);
        std::unique_ptr<Dev> pg[7];
        const int64_t psz[7] = {int64_t(heads) * dp(), int64_t(heads) * dp(), heads * 2 * int64_t(hidden),
                                int64_t(heads) * hidden, int64_t(heads) * hidden, heads, heads};
        for (int i = 0; i < 7; ++i) {
            pg[i] = std::make_unique<Dev>(psz[i] * 4);
            ccheck(cudaMemset(pg[i]->p, 0, psz[i] * 4), "memset");
        }
        affmae_attn_grads g{dq.as<affmae_bf16>(), dk.as<affmae_bf16>(), dv.as<affmae_bf16>(),
                            pg[0]->as<float>(), pg[1]->as<float>(), pg[2]->as<float>(), pg[3]->as<float>(),
                            pg[4]->as<float>(), pg[5]->as<float>(), pg[6]->as<float>()};
        Dev wsb(affmae_attn_bwd_planned_workspace(&G.d.g, &a));
        check(affmae_attn_bwd_planned(&G.d.g, &a, &S.ai, &G.plan, S.out->as<affmae_bf16>(), S.lse->as<float>(),
                                      dout->as<affmae_bf16>(), &g, wsb.p, wsb.n, nullptr),
              "attn_bwd");
        ccheck(cudaDeviceSynchronize(), "sync");
        // accumulate (+=) into non-null in_grads (include/affmae/tape.hpp:29-31), padded columns dropped
        const Dev* act[3] = {&dq, &dk, &dv};
        const float sc[3] = {qscale(), 1.f, 1.f};
        for (int i = 0; i < 3; ++i) {
            if (!in_grads[size_t(i)]) continue;
            auto h = download<uint16_t>(*act[i], size_t(n * hd));
            for (int64_t r = 0; r < n; ++r)
                for (int gq = 0; gq < heads; ++gq)
                    for (int e = 0; e < head_dim; ++e) {
                        const int64_t j = (r * heads + gq) * head_dim + e;
                        in_grads[size_t(i)]->set(j, in_grads[size_t(i)]->get(j) +
                                                        sc[i] * bf16_to_float(h[size_t(pad_at(r, gq, e, heads, dp()))]));
                    }
        }
        for (int i = 0; i < 7; ++i) {
            Tensor* dst = in_grads[size_t(3 + i)];
            if (!dst) continue;
            auto h = download<float>(*pg[i], size_t(psz[i]));
            if (i < 2) {  // blank rows [heads, dp] -> [heads, head_dim]
                for (int gq = 0; gq < heads; ++gq)
                    for (int e = 0; e < head_dim; ++e)
                        dst->set(gq * head_dim + e, dst->get(gq * head_dim + e) + h[size_t(gq * dp() + e)]);
                continue;
            }
            for (int64_t j = 0; j < psz[i]; ++j) dst->set(j, dst->get(j) + h[size_t(j)]);
        }
    }
};

}  // namespace

std::shared_ptr<CustomOp> make_cluster_attn_op(Tensor coords, int64_t cluster, int64_t groups, int heads,
                                               int head_dim, int bias_hidden, double patch) {
    auto op = std::make_shared<ClusterAttnOp>();
    op->coords = std::move(coords);
    op->cluster = cluster;
    op->groups = groups;
    op->heads = heads;
    op->head_dim = head_dim;
    op->hidden = bias_hidden;
    op->patch = patch;
    return op;
}

std::vector<int64_t> select_retained(const Tensor& scores, double d_s) {
    const int64_t n = scores.rows();
    const int64_t r = affmae_retained_count(n, d_s);
    if (r < 0) throw ConfigError("retained_count: d_s must be in (0, 1]");
    auto s = upload(f32(scores));
    Dev out(r * 4), ws(affmae_select_retained_workspace(1, n));
    check(affmae_select_retained(s->as<float>(), 1, n, d_s, out.as<int32_t>(), ws.p, ws.n, nullptr), "select_retained");
    auto h = download<int32_t>(out, size_t(r));
    return std::vector<int64_t>(h.begin(), h.end());
}

MergePlan merge_plan(const PointSet& ps, std::span<const int64_t> retained, int k_m) {
    const int64_t n = ps.count(), r = int64_t(retained.size());
    if (r < 1) throw ConfigError("merge_plan: retained set empty");
    auto c = upload(f32(ps.coords));
    std::vector<int32_t> rv(retained.begin(), retained.end());
    auto dr = upload(rv);
    Dev tgt(n * 4), pidx(r * k_m * 4), pdist(r * k_m * 8), pcnt(r * 4), rowof(n * 4),
        ws(affmae_merge_plan_workspace(1, n, r));
    affmae_merge_plan pl{tgt.as<int32_t>(), pidx.as<int32_t>(), pdist.as<double>(), pcnt.as<int32_t>(),
                         rowof.as<int32_t>()};
    check(affmae_merge_plan_build(c->as<float>(), dr->as<int32_t>(), 1, n, r, k_m, &pl, ws.p, ws.n, nullptr),
          "merge_plan");
    auto ht = download<int32_t>(tgt, size_t(n));
    auto hi = download<int32_t>(pidx, size_t(r * k_m));
    auto hd = download<double>(pdist, size_t(r * k_m));
    auto hc = download<int32_t>(pcnt, size_t(r));
    MergePlan plan;
    plan.retained.assign(retained.begin(), retained.end());
    for (int64_t j = 0; j < n; ++j)
        if (ht[size_t(j)] >= 0) {
            plan.dropped.push_back(j);
            plan.target.push_back(ht[size_t(j)]);
        }
    plan.pool.resize(size_t(r));
    plan.pool_dist.resize(size_t(r));
    for (int64_t i = 0; i < r; ++i)
        for (int t = 0; t < hc[size_t(i)]; ++t) {
            plan.pool[size_t(i)].push_back(hi[size_t(i * k_m + t)]);
            plan.pool_dist[size_t(i)].push_back(hd[size_t(i * k_m + t)]);
        }
    return plan;
}

std::shared_ptr<CustomOp> make_merge_pool_op(MergePlan plan) {
    // The device pool kernels consume the device plan; rebuild it from the host plan.
    struct PoolOp final : CustomOp {
        MergePlan plan;
        std::string name() const override { return "merge_pool_b200"; }
        int km() const {
            size_t m = 1;
            for (auto& p : plan.pool) m = std::max(m, p.size());
            return int(m);
        }
        struct DevPlan {
            std::unique_ptr<Dev> ret, tgt, pidx, pdist, pcnt, rowof;
            affmae_merge_plan pl{};
        };
        DevPlan upload_plan(int64_t n, int k_m) const {
            const int64_t r = int64_t(plan.retained.size());
            std::vector<int32_t> ret(plan.retained.begin(), plan.retained.end());
            std::vector<int32_t> tgt(static_cast<size_t>(n), -1), rowof(static_cast<size_t>(n), -1);
            std::vector<int32_t> pidx(static_cast<size_t>(r * k_m), -1), pcnt(static_cast<size_t>(r), 0);
            std::vector<double> pdist(static_cast<size_t>(r * k_m), 0.0);
            for (size_t i = 0; i < plan.dropped.size(); ++i) tgt[size_t(plan.dropped[i])] = int32_t(plan.target[i]);
            for (int64_t i = 0; i < r; ++i) {
                rowof[size_t(plan.retained[size_t(i)])] = int32_t(i);
                pcnt[size_t(i)] = int32_t(plan.pool[size_t(i)].size());
                for (size_t t = 0; t < plan.pool[size_t(i)].size(); ++t) {
                    pidx[size_t(i * k_m) + t] = int32_t(plan.pool[size_t(i)][t]);
                    pdist[size_t(i * k_m) + t] = plan.pool_dist[size_t(i)][t];
                    rowof[size_t(plan.pool[size_t(i)][t])] = int32_t(i);
                }
            }
            DevPlan d;
            d.ret = upload(ret);
            d.tgt = upload(tgt);
            d.pidx = upload(pidx);
            d.pdist = upload(pdist);
            d.pcnt = upload(pcnt);
            d.rowof = upload(rowof);
            d.pl = {d.tgt->as<int32_t>(), d.pidx->as<int32_t>(), d.pdist->as<double>(), d.pcnt->as<int32_t>(),
                    d.rowof->as<int32_t>()};
            return d;
        }
        Tensor forward(const std::vector<const Tensor*>& in) override {
            const Tensor& feats = *in[0];
            const int64_t n = feats.rows(), dim = feats.cols(), r = int64_t(plan.retained.size());
            const int k_m = km();
            DevPlan d = upload_plan(n, k_m);
            auto f = upload(bf16(feats));
            auto s = upload(f32(*in[1]));
            auto pm = upload(f32(*in[2]));
            Dev out(r * 2 * dim * 2);
            check(affmae_merge_pool_fwd(f->as<affmae_bf16>(), s->as<float>(), pm->as<float>(), d.ret->as<int32_t>(),
                                        &d.pl, 1, n, r, dim, k_m, out.as<affmae_bf16>(), nullptr), "merge_pool_fwd");
            auto h = download<uint16_t>(out, size_t(r * 2 * dim));
            Tensor o = Tensor::zeros({r, 2 * dim}, feats.precision());
            for (int64_t i = 0; i < r * 2 * dim; ++i) o.set(i, bf16_to_float(h[size_t(i)]));
            return o;
        }
        void backward(const Tensor& g, const std::vector<const Tensor*>& in,
                      const std::vector<Tensor*>& in_grads) override {
            const Tensor& feats = *in[0];
            const int64_t n = feats.rows(), dim = feats.cols(), r = int64_t(plan.retained.size());
            const int k_m = km();
            DevPlan d = upload_plan(n, k_m);
            auto f = upload(bf16(feats));
            auto s = upload(f32(*in[1]));
            auto pm = upload(f32(*in[2]));
            auto dg = upload(bf16(g));
            Dev df(n * dim * 2), ds(n * 4), dp(4), ws(affmae_merge_pool_bwd_workspace(1, r));
            ccheck(cudaMemset(dp.p, 0, 4), "memset");
            check(affmae_merge_pool_bwd(f->as<affmae_bf16>(), s->as<float>(), pm->as<float>(), d.ret->as<int32_t>(),
                                        &d.pl, 1, n, r, dim, k_m, dg->as<affmae_bf16>(), df.as<affmae_bf16>(),
                                        ds.as<float>(), dp.as<float>(), ws.p, ws.n, nullptr), "merge_pool_bwd");
            if (in_grads[0]) {
                auto h = download<uint16_t>(df, size_t(n * dim));
                for (int64_t i = 0; i < n * dim; ++i) in_grads[0]->set(i, in_grads[0]->get(i) + bf16_to_float(h[size_t(i)]));
            }
            if (in_grads[1]) {
                auto h = download<float>(ds, size_t(n));
                for (int64_t i = 0; i < n; ++i) in_grads[1]->set(i, in_grads[1]->get(i) + h[size_t(i)]);
            }
            if (in_grads[2]) in_grads[2]->set(0, in_grads[2]->get(0) + download<float>(dp, 1)[0]);
        }
    };
    auto op = std::make_shared<PoolOp>();
    op->plan = std::move(plan);
    return op;
}

std::shared_ptr<CustomOp> make_interp_op(Tensor key_coords, NeighborIndex nbrs, double eps) {
    struct InterpCudaOp final : CustomOp {
        Tensor key_coords;
        NeighborIndex nbrs;
        double eps = kInterpEps;
        std::string name() const override { return "interp_softmax_b200"; }
        struct DevRows {
            std::unique_ptr<Dev> kc, idx, valid;
        };
        DevRows upload_rows() const {
            if (nbrs.width < 1 || nbrs.width > 32) throw ConfigError("interp op: neighbour width must be in [1, 32]");
            std::vector<int32_t> idx(nbrs.idx.begin(), nbrs.idx.end());
            DevRows d;
            d.kc = upload(f32(key_coords));
            d.idx = upload(idx);
            d.valid = upload(nbrs.valid);
            return d;
        }
        void validate(const Tensor& feats, const Tensor& pt, const Tensor& q) const {
            if (pt.numel() != 1) throw ConfigError("interp op: p must be scalar");
            if (q.ndim() != 2 || q.dim(1) != 2) throw ConfigError("interp op: queries must be Qx2");
            if (q.dim(0) != nbrs.queries()) throw ConfigError("interp op: query count does not match neighbor index");
            for (int64_t qi = 0; qi < nbrs.queries(); ++qi)
                if (nbrs.row(qi).empty()) throw ConfigError("interp_softmax: no valid neighbors");
            (void)feats;
        }
        // feature widths the kernels are not compiled for run zero-padded to the next of 64..512
        static int64_t padded(int64_t dim) {
            for (int64_t w : {64, 128, 256, 512})
                if (dim <= w) return w;
            throw ConfigError("interp op: feature width > 512 not compiled");
        }
        Tensor forward(const std::vector<const Tensor*>& in) override {
            const Tensor& feats = *in[0];
            validate(feats, *in[1], *in[2]);
            const int64_t nk = feats.rows(), dim0 = feats.cols(), dim = padded(dim0), nq = in[2]->dim(0);
            DevRows d = upload_rows();
            auto f = upload(bf16_pad(feats, 1, dim0, dim));
            auto pt = upload(f32(*in[1]));
            auto q = upload(f32(*in[2]));
            Dev out(nq * dim * 2);
            check(affmae_interp_fwd(q->as<float>(), d.kc->as<float>(), f->as<affmae_bf16>(), d.idx->as<int32_t>(),
                                    d.valid->as<uint8_t>(), 1, nq, nk, dim, nbrs.width, pt->as<float>(), eps,
                                    out.as<affmae_bf16>(), nullptr),
                  "interp_fwd");
            auto h = download<uint16_t>(out, size_t(nq * dim));
            Tensor o = Tensor::zeros({nq, dim0}, feats.precision());
            for (int64_t r = 0; r < nq; ++r)
                for (int64_t e = 0; e < dim0; ++e) o.set(r * dim0 + e, bf16_to_float(h[size_t(r * dim + e)]));
            return o;
        }
        void backward(const Tensor& g, const std::vector<const Tensor*>& in,
                      const std::vector<Tensor*>& in_grads) override {
            const Tensor& feats = *in[0];
            const int64_t nk = feats.rows(), dim0 = feats.cols(), dim = padded(dim0), nq = in[2]->dim(0);
            DevRows d = upload_rows();
            auto f = upload(bf16_pad(feats, 1, dim0, dim));
            auto pt = upload(f32(*in[1]));
            auto q = upload(f32(*in[2]));
            auto dg = upload(bf16_pad(g, 1, dim0, dim));
            Dev df(nk * dim * 4), dp(4), dq(nq * 2 * 4);
            ccheck(cudaMemset(df.p, 0, size_t(nk * dim * 4)), "memset");
            ccheck(cudaMemset(dp.p, 0, 4), "memset");
            ccheck(cudaMemset(dq.p, 0, size_t(nq * 2 * 4)), "memset");
            Dev ws(affmae_interp_bwd_gather_workspace(1, nq, nk, nbrs.width));
            check(affmae_interp_bwd_gather(q->as<float>(), d.kc->as<float>(), f->as<affmae_bf16>(),
                                           d.idx->as<int32_t>(), d.valid->as<uint8_t>(), 1, nq, nk, dim, nbrs.width,
                                           pt->as<float>(), eps, dg->as<affmae_bf16>(), df.as<float>(), dp.as<float>(),
                                           dq.as<float>(), ws.p, ws.n, nullptr),
                  "interp_bwd");
            if (in_grads[0]) {
                auto h = download<float>(df, size_t(nk * dim));
                for (int64_t r = 0; r < nk; ++r)
                    for (int64_t e = 0; e < dim0; ++e)
                        in_grads[0]->set(r * dim0 + e, in_grads[0]->get(r * dim0 + e) + h[size_t(r * dim + e)]);
            }
            if (in_grads[1]) in_grads[1]->set(0, in_grads[1]->get(0) + download<float>(dp, 1)[0]);
            if (in_grads[2]) {
                auto h = download<float>(dq, size_t(nq * 2));
                for (int64_t i = 0; i < nq * 2; ++i) in_grads[2]->set(i, in_grads[2]->get(i) + h[size_t(i)]);
            }
        }
    };
    auto op = std::make_shared<InterpCudaOp>();
    op->key_coords = std::move(key_coords);
    op->nbrs = std::move(nbrs);
    op->eps = eps;
    return op;
}

// Attention over a general NeighborIndex: the decoder's cross (one_to_one) and self (knn)
// attention layers.  Rows of width <= 31.
std::shared_ptr<CustomOp> make_general_attn_op(Tensor coords, NeighborIndex nbr, int heads, int head_dim,
                                               int bias_hidden, double patch) {
    struct GAttnCudaOp final : CustomOp {
        Tensor coords;
        NeighborIndex nbr;
        int heads, head_dim, hidden;
        double patch;
        std::string name() const override { return "nbhd_attention_b200"; }
        int dp() const { return padded_head_dim(head_dim); }
        float qscale() const { return float(std::sqrt(double(dp()) / double(head_dim))); }
        struct Up {
            std::unique_ptr<Dev> t[10], coords, idx, valid;
            affmae_attn_inputs ai{};
        };
        Up upload_all(const std::vector<const Tensor*>& in) const {
            if (in.size() != 10) throw ConfigError("attention op: want 10 inputs");
            if (nbr.width < 1 || nbr.width > 31) throw ConfigError("attention op: neighbour width must be in [1, 31]");
            if (in[0]->rows() != nbr.queries()) throw ConfigError("attention op: row count does not match neighbor index");
            Up u;
            u.t[0] = upload(bf16_pad(*in[0], heads, head_dim, dp(), qscale()));
            for (int i = 1; i < 3; ++i) u.t[i] = upload(bf16_pad(*in[size_t(i)], heads, head_dim, dp()));
            for (int i = 3; i < 5; ++i) u.t[i] = upload(bf16_pad(*in[size_t(i)], 1, head_dim, dp()));
            for (int i = 5; i < 10; ++i) u.t[i] = upload(f32(*in[size_t(i)]));
            u.coords = upload(f32(coords));
            std::vector<int32_t> idx(nbr.idx.begin(), nbr.idx.end());
            u.idx = upload(idx);
            u.valid = upload(nbr.valid);
            u.ai = {u.t[0]->as<affmae_bf16>(), u.t[1]->as<affmae_bf16>(), u.t[2]->as<affmae_bf16>(),
                    u.t[3]->as<affmae_bf16>(), u.t[4]->as<affmae_bf16>(), u.coords->as<float>(),
                    u.t[5]->as<float>(), u.t[6]->as<float>(), u.t[7]->as<float>(), u.t[8]->as<float>(),
                    u.t[9]->as<float>()};
            return u;
        }
        Tensor forward(const std::vector<const Tensor*>& in) override {
            Up u = upload_all(in);
            const int64_t n = in[0]->rows(), hd = int64_t(heads) * head_dim, hdp = int64_t(heads) * dp();
            affmae_attn_desc a{heads, dp(), hidden, patch};
            Dev out(n * hdp * 2), lse(n * heads * 4);
            check(affmae_gattn_fwd(&a, &u.ai, u.idx->as<int32_t>(), u.valid->as<uint8_t>(), 1, n, nbr.width,
                                   out.as<affmae_bf16>(), lse.as<float>(), nullptr),
                  "gattn_fwd");
            auto h = download<uint16_t>(out, size_t(n * hdp));
            Tensor o = Tensor::zeros({n, hd}, in[0]->precision());
            for (int64_t r = 0; r < n; ++r)
                for (int g = 0; g < heads; ++g)
                    for (int e = 0; e < head_dim; ++e)
                        o.set((r * heads + g) * head_dim + e, bf16_to_float(h[size_t(pad_at(r, g, e, heads, dp()))]));
            return o;
        }
        void backward(const Tensor& out_grad, const std::vector<const Tensor*>& in,
                      const std::vector<Tensor*>& in_grads) override {
            Up u = upload_all(in);
            const int64_t n = in[0]->rows(), hdp = int64_t(heads) * dp();
            affmae_attn_desc a{heads, dp(), hidden, patch};
            auto dout = upload(bf16_pad(out_grad, heads, head_dim, dp()));
            const int64_t sz[10] = {n * hdp, n * hdp, n * hdp, int64_t(heads) * dp(), int64_t(heads) * dp(),
                                    heads * 2 * int64_t(hidden), int64_t(heads) * hidden, int64_t(heads) * hidden,
                                    heads, heads};
            Dev dq(n * hdp * 2);
            std::unique_ptr<Dev> g[10];
            for (int i = 1; i < 10; ++i) {
                g[i] = std::make_unique<Dev>(sz[i] * 4);
                ccheck(cudaMemset(g[i]->p, 0, size_t(sz[i] * 4)), "memset");
            }
            check(affmae_gattn_bwd(&a, &u.ai, u.idx->as<int32_t>(), u.valid->as<uint8_t>(), 1, n, nbr.width,
                                   dout->as<affmae_bf16>(), dq.as<affmae_bf16>(), g[1]->as<float>(),
                                   g[2]->as<float>(), g[3]->as<float>(), g[4]->as<float>(), g[5]->as<float>(),
                                   g[6]->as<float>(), g[7]->as<float>(), g[8]->as<float>(), g[9]->as<float>(),
                                   nullptr, 0, nullptr),
                  "gattn_bwd");
            ccheck(cudaDeviceSynchronize(), "sync");
            auto put_rows = [&](Tensor* dst, const std::vector<float>& h, int64_t rows, int64_t groups, float sc) {
                for (int64_t r = 0; r < rows; ++r)
                    for (int64_t gq = 0; gq < groups; ++gq)
                        for (int e = 0; e < head_dim; ++e) {
                            const int64_t j = (r * groups + gq) * head_dim + e;
                            dst->set(j, dst->get(j) + sc * h[size_t(pad_at(r, gq, e, groups, dp()))]);
                        }
            };
            if (in_grads[0]) {
                auto h = download<uint16_t>(dq, size_t(n * hdp));
                std::vector<float> f(h.size());
                for (size_t j = 0; j < h.size(); ++j) f[j] = bf16_to_float(h[j]);
                put_rows(in_grads[0], f, n, heads, qscale());
            }
            for (int i = 1; i < 10; ++i) {
                Tensor* dst = in_grads[size_t(i)];
                if (!dst) continue;
                auto h = download<float>(*g[i], size_t(sz[i]));
                if (i <= 2) put_rows(dst, h, n, heads, 1.f);
                else if (i <= 4) put_rows(dst, h, heads, 1, 1.f);
                else
                    for (int64_t j = 0; j < sz[i]; ++j) dst->set(j, dst->get(j) + h[size_t(j)]);
            }
        }
    };
    auto op = std::make_shared<GAttnCudaOp>();
    op->coords = std::move(coords);
    op->nbr = std::move(nbr);
    op->heads = heads;
    op->head_dim = head_dim;
    op->hidden = bias_hidden;
    op->patch = patch;
    return op;
}

// The (cluster size, groups) whose cluster_neighborhood (src/geometry.cpp:133-186) on `coords`
// is exactly `nbr`, if any: the NeighborIndex rebuilt on the device for every (size, groups)
// consistent with its width (width = groups_eff * ceil(n / C)) and compared entry for entry.
bool detect_cluster_index(const Tensor& coords, const NeighborIndex& nbr, int64_t* size_out, int64_t* groups_out) {
    const int64_t n = nbr.queries(), m = nbr.width;
    if (n < 1 || m < 1 || coords.rows() != n) return false;
    auto c = upload(f32(coords));
    for (int64_t g = 1; g <= m; ++g) {
        if (m % g) continue;
        const int64_t mx = m / g;  // largest cluster
        if (mx > 16) continue;     // compiled cluster kernels
        for (int64_t s = mx; s <= 2 * mx + 1; ++s) {
            affmae_cluster_geom geo{1, n, s, g, 0, 0, 0, 0};
            if (affmae_cluster_geometry(&geo) != AFFMAE_OK || geo.width != m || geo.groups_eff != g) continue;
            DeviceIndex d = build_index(*c, n, s, g);
            Dev idx(n * m * 4), valid(n * m);
            check(affmae_neighbor_expand(&d.g, d.perm->as<int32_t>(), d.nbr->as<int32_t>(), idx.as<int32_t>(),
                                         valid.as<uint8_t>(), nullptr), "neighbor_expand");
            ccheck(cudaDeviceSynchronize(), "sync");
            auto hi = download<int32_t>(idx, size_t(n * m));
            auto hv = download<uint8_t>(valid, size_t(n * m));
            bool same = true;
            for (size_t e = 0; same && e < hi.size(); ++e)
                same = (hv[e] != 0) == (nbr.valid[e] != 0) && (!hv[e] || int64_t(hi[e]) == nbr.idx[e]);
            if (same) {
                *size_out = s;
                *groups_out = g;
                return true;
            }
        }
    }
    return false;
}

std::shared_ptr<CustomOp> make_attn_op(Tensor coords, NeighborIndex nbr, int heads, int head_dim, int bias_hidden,
                                       double patch, bool streaming, bool half_io) {
    (void)streaming;  // the device kernels are the streaming (online softmax) formulation
    (void)half_io;    // activations are bf16 on the device either way
    int64_t size = 0, groups = 0;
    if (detect_cluster_index(coords, nbr, &size, &groups))
        return make_cluster_attn_op(std::move(coords), size, groups, heads, head_dim, bias_hidden, patch);
    if (nbr.width <= 31) return make_general_attn_op(std::move(coords), std::move(nbr), heads, head_dim, bias_hidden, patch);
    throw ConfigError("cuda::make_attn_op: neighbour rows wider than 31 must be a cluster_neighborhood index");
}

MaskSpec perlin_mask(int64_t hp, int64_t wp, double ratio, uint64_t seed) {
    if (hp != wp) throw ConfigError("cuda::perlin_mask: square grids only");
    Dev ws(affmae_perlin_mask_workspace(1, hp, wp, kPerlinOctaves, kPerlinBaseFreq)), out(size_t(hp * wp));
    check(affmae_perlin_mask(&seed, 1, hp, wp, kPerlinOctaves, kPerlinBaseFreq, kPerlinPersistence, ratio,
                             out.as<uint8_t>(), ws.p, ws.n, nullptr),
          "perlin_mask");
    MaskSpec m;  // as mask_from_field fills it (src/masking.cpp:71-92)
    m.hp = hp;
    m.wp = wp;
    m.ratio = ratio;
    m.masked = download<uint8_t>(out, size_t(hp * wp));
    return m;
}

Tensor synth_image(int64_t size, uint64_t seed) {
    Dev ws(affmae_synth_images_workspace(1, size)), img(size_t(size * size) * 8);
    check(affmae_synth_images(&seed, 1, size, img.as<double>(), ws.p, ws.n, nullptr), "synth_image");
    auto h = download<double>(img, size_t(size * size));
    Tensor t = Tensor::zeros({size, size}, Precision::b64);
    for (int64_t i = 0; i < size * size; ++i) t.set(i, h[size_t(i)]);
    return t;
}

}  // namespace affmae::cuda
