// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python tests, the golden-vector generator and bench.py's CPU legs call
// the reference's own hot-path functions on plain arrays:
//
//   ref_sfc_order            -> affmae::sfc_order            (proj/src/geometry.cpp:69-106)
//   ref_cluster_index        -> balanced_clusters + cluster_neighborhood (geometry.cpp:108-186)
//   ref_knn                  -> affmae::knn                  (geometry.cpp:188-216)
//   ref_attn_fwd             -> nbhd_attn_streaming / _naive (proj/src/attention.cpp:189-220)
//   ref_attn_bwd             -> nbhd_attn_backward           (attention.cpp:241-358)
//   ref_select_retained      -> select_retained              (proj/src/merging.cpp:56-69)
//   ref_merge_plan           -> merge_plan                   (merging.cpp:71-116)
//   ref_merge_pool_fwd/bwd   -> make_merge_pool_op forward/backward (merging.cpp:151-220)
//   ref_perlin_mask          -> perlin_field + mask_from_field (proj/src/masking.cpp:51-92)
//   ref_synth_image          -> synth_image                  (proj/src/pipeline.cpp:169-227)
//   ref_write_aft / _u8, ref_read_aft -> write_aft / write_aft_u8 / read_aft (proj/src/tensor_io.cpp:60-105)
//   ref_hotpath_batch        -> the whole hot path over B images on T std::threads
//                               (the multi-core CPU baseline of BASELINE.md §4)
//
// All functions return 0 on success, 2 on ConfigError, 3 on NumericError,
// 1 on anything else; the message is kept in ref_last_error().
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "affmae/attention.hpp"
#include "affmae/errors.hpp"
#include "affmae/geometry.hpp"
#include "affmae/interpolation.hpp"
#include "affmae/masking.hpp"
#include "affmae/merging.hpp"
#include "affmae/pipeline.hpp"
#include "affmae/tape.hpp"
#include "affmae/tensor.hpp"
#include "affmae/tensor_io.hpp"

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

Precision prec_of(int p) { return p == 64 ? Precision::b64 : Precision::b32; }

Tensor from(const double* p, std::vector<int64_t> dims, Precision prec) {
    Tensor t = Tensor::zeros(std::move(dims), prec);
    for (int64_t i = 0; i < t.numel(); ++i) t.set(i, p[i]);
    return t;
}
Tensor from_f(const float* p, std::vector<int64_t> dims, Precision prec) {
    Tensor t = Tensor::zeros(std::move(dims), prec);
    for (int64_t i = 0; i < t.numel(); ++i) t.set(i, double(p[i]));
    return t;
}
void to(const Tensor& t, double* out) {
    for (int64_t i = 0; i < t.numel(); ++i) out[i] = t.get(i);
}

PointSet points(const float* coords, int64_t n) {
    PointSet ps;
    ps.coords = from_f(coords, {n, 2}, Precision::b32);
    ps.feats = Tensor::zeros({n, 0}, Precision::b32);
    return ps;
}

NeighborIndex nbr_from(const int64_t* idx, const uint8_t* valid, int64_t n, int64_t m) {
    NeighborIndex nb;
    nb.width = m;
    nb.idx.assign(idx, idx + n * m);
    nb.valid.assign(valid, valid + n * m);
    return nb;
}

struct AttnInputs {
    Tensor q, k, v, bk, bv, coords;
    NeighborIndex nbr;
    BiasNet bias;
    AttnCtx ctx(int heads, int d) const {
        AttnCtx c;
        c.q = &q;
        c.k = &k;
        c.v = &v;
        c.blank_k = &bk;
        c.blank_v = &bv;
        c.coords = &coords;
        c.nbr = &nbr;
        c.bias = &bias;
        c.heads = heads;
        c.head_dim = d;
        return c;
    }
};

AttnInputs attn_inputs(int64_t n, int64_t m, int heads, int d, int hidden, double patch,
                       const double* q, const double* k, const double* v, const double* bk,
                       const double* bv, const float* coords, const int64_t* idx,
                       const uint8_t* valid, const double* w1, const double* b1,
                       const double* w2, const double* b2, const double* blank, Precision prec) {
    AttnInputs a;
    int64_t hd = int64_t(heads) * d;
    a.q = from(q, {n, hd}, prec);
    a.k = from(k, {n, hd}, prec);
    a.v = from(v, {n, hd}, prec);
    a.bk = from(bk, {heads, d}, prec);
    a.bv = from(bv, {heads, d}, prec);
    a.coords = from_f(coords, {n, 2}, Precision::b32);
    a.nbr = nbr_from(idx, valid, n, m);
    a.bias.heads = heads;
    a.bias.hidden = hidden;
    a.bias.patch = patch;
    a.bias.w1 = from(w1, {heads, 2 * hidden}, prec);
    a.bias.b1 = from(b1, {heads, hidden}, prec);
    a.bias.w2 = from(w2, {heads, hidden}, prec);
    a.bias.b2 = from(b2, {heads, 1}, prec);
    a.bias.blank = from(blank, {heads, 1}, prec);
    return a;
}

MergePlan plan_from(int64_t r, int k_m, const int64_t* retained, const int64_t* pool_idx,
                    const double* pool_dist, const int32_t* pool_cnt) {
    MergePlan plan;
    plan.retained.assign(retained, retained + r);
    plan.pool.resize(size_t(r));
    plan.pool_dist.resize(size_t(r));
    for (int64_t i = 0; i < r; ++i)
        for (int32_t t = 0; t < pool_cnt[i]; ++t) {
            plan.pool[size_t(i)].push_back(pool_idx[i * k_m + t]);
            plan.pool_dist[size_t(i)].push_back(pool_dist[i * k_m + t]);
        }
    return plan;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_sfc_order(const float* coords, int64_t n, int64_t* perm) {
    return guarded([&] {
        std::vector<int64_t> p = sfc_order(points(coords, n));
        std::memcpy(perm, p.data(), p.size() * sizeof(int64_t));
    });
}

// Geometry of balanced_clusters/cluster_neighborhood without running them.
int ref_cluster_shape(int64_t n, int64_t size, int64_t groups, int64_t* n_clusters,
                      int64_t* groups_eff, int64_t* max_size, int64_t* width) {
    return guarded([&] {
        if (size < 1 || groups < 1 || n < 1) throw ConfigError("bad shape");
        int64_t s = std::min(size, n);
        int64_t c = (n + s - 1) / s;
        *n_clusters = c;
        *groups_eff = std::min(groups, c);
        *max_size = n / c + (n % c ? 1 : 0);
        *width = *groups_eff * *max_size;
    });
}

// cluster_of [n]; members [n] (curve order, cluster-major); member_off [c+1];
// idx/valid [n * width]
int ref_cluster_index(const float* coords, int64_t n, int64_t size, int64_t groups,
                      int32_t* cluster_of, int64_t* members, int64_t* member_off, int64_t* idx,
                      uint8_t* valid, int64_t width_cap) {
    return guarded([&] {
        PointSet ps = points(coords, n);
        ClusterAssignment a = balanced_clusters(ps, size);
        NeighborIndex nb = cluster_neighborhood(a, ps, groups);
        if (nb.width > width_cap) throw ConfigError("width_cap too small");
        std::memcpy(cluster_of, a.cluster_of.data(), size_t(n) * sizeof(int32_t));
        int64_t pos = 0;
        member_off[0] = 0;
        for (int64_t c = 0; c < a.count(); ++c) {
            for (int64_t t : a.members[size_t(c)]) members[pos++] = t;
            member_off[c + 1] = pos;
        }
        for (int64_t q = 0; q < n; ++q)
            for (int64_t m = 0; m < width_cap; ++m) {
                bool in = m < nb.width;
                idx[q * width_cap + m] = in ? nb.key(q, m) : 0;
                valid[q * width_cap + m] = in ? nb.valid[size_t(q * nb.width + m)] : 0;
            }
    });
}

int ref_knn(const float* queries, int64_t nq, const float* keys, int64_t nk, int64_t k,
            int64_t* idx, uint8_t* valid) {
    return guarded([&] {
        Tensor q = from_f(queries, {nq, 2}, Precision::b32);
        NeighborIndex nb = knn(q, points(keys, nk), k);
        std::memcpy(idx, nb.idx.data(), nb.idx.size() * sizeof(int64_t));
        std::memcpy(valid, nb.valid.data(), nb.valid.size());
    });
}

// prec: 32 or 64 (tensor precision of q/k/v/blanks/bias); mode: 0 streaming,
// 1 naive, 2 streaming with half_io.
int ref_attn_fwd(int64_t n, int64_t m, int heads, int d, int hidden, double patch, const double* q,
                 const double* k, const double* v, const double* bk, const double* bv,
                 const float* coords, const int64_t* idx, const uint8_t* valid, const double* w1,
                 const double* b1, const double* w2, const double* b2, const double* blank,
                 int prec, int mode, double* out) {
    return guarded([&] {
        AttnInputs a = attn_inputs(n, m, heads, d, hidden, patch, q, k, v, bk, bv, coords, idx,
                                   valid, w1, b1, w2, b2, blank, prec_of(prec));
        AttnCtx c = a.ctx(heads, d);
        Tensor o = mode == 1 ? nbhd_attn_naive(c) : nbhd_attn_streaming(c, mode == 2);
        to(o, out);
    });
}

int ref_attn_bwd(int64_t n, int64_t m, int heads, int d, int hidden, double patch, const double* q,
                 const double* k, const double* v, const double* bk, const double* bv,
                 const float* coords, const int64_t* idx, const uint8_t* valid, const double* w1,
                 const double* b1, const double* w2, const double* b2, const double* blank,
                 int prec, const double* dout, double* dq, double* dk, double* dv, double* dbk,
                 double* dbv, double* dw1, double* db1, double* dw2, double* db2,
                 double* dblank) {
    return guarded([&] {
        AttnInputs a = attn_inputs(n, m, heads, d, hidden, patch, q, k, v, bk, bv, coords, idx,
                                   valid, w1, b1, w2, b2, blank, prec_of(prec));
        int64_t hd = int64_t(heads) * d;
        Tensor cot = from(dout, {n, hd}, prec_of(prec));
        AttnGrads g = nbhd_attn_backward(a.ctx(heads, d), cot);
        to(g.dq, dq);
        to(g.dk, dk);
        to(g.dv, dv);
        to(g.dblank_k, dbk);
        to(g.dblank_v, dbv);
        to(g.dw1, dw1);
        to(g.db1, db1);
        to(g.dw2, dw2);
        to(g.db2, db2);
        to(g.dblank, dblank);
    });
}

int64_t ref_retained_count(int64_t n, double d_s) {
    int64_t out = -1;
    if (guarded([&] { out = retained_count(n, d_s); })) return -1;
    return out;
}

int ref_select_retained(const double* scores, int64_t n, double d_s, int prec, int64_t* out,
                        int64_t* n_out) {
    return guarded([&] {
        std::vector<int64_t> r = select_retained(from(scores, {n, 1}, prec_of(prec)), d_s);
        std::memcpy(out, r.data(), r.size() * sizeof(int64_t));
        *n_out = int64_t(r.size());
    });
}

// dropped/target: [n - r] in ascending dropped order; pool_idx/pool_dist:
// [r * k_m] (first pool_cnt[i] valid)
int ref_merge_plan(const float* coords, int64_t n, const int64_t* retained, int64_t r, int k_m,
                   int64_t* dropped, int64_t* target, int64_t* pool_idx, double* pool_dist,
                   int32_t* pool_cnt) {
    return guarded([&] {
        MergePlan plan = merge_plan(points(coords, n), std::span<const int64_t>(retained, size_t(r)), k_m);
        for (size_t i = 0; i < plan.dropped.size(); ++i) {
            dropped[i] = plan.dropped[i];
            target[i] = plan.target[i];
        }
        for (int64_t i = 0; i < r; ++i) {
            const auto& p = plan.pool[size_t(i)];
            pool_cnt[i] = int32_t(p.size());
            for (size_t t = 0; t < size_t(k_m); ++t) {
                pool_idx[i * k_m + int64_t(t)] = t < p.size() ? p[t] : -1;
                pool_dist[i * k_m + int64_t(t)] = t < p.size() ? plan.pool_dist[size_t(i)][t] : 0.0;
            }
        }
    });
}

int ref_merge_pool_fwd(int64_t n, int64_t dim, int64_t r, int k_m, const int64_t* retained,
                       const int64_t* pool_idx, const double* pool_dist, const int32_t* pool_cnt,
                       const double* feats, const double* scores, double p, int prec,
                       double* out) {
    return guarded([&] {
        auto op = make_merge_pool_op(plan_from(r, k_m, retained, pool_idx, pool_dist, pool_cnt));
        Tensor f = from(feats, {n, dim}, prec_of(prec));
        Tensor s = from(scores, {n, 1}, prec_of(prec));
        Tensor pt = Tensor::full({1, 1}, p, prec_of(prec));
        Tensor o = op->forward({&f, &s, &pt});
        to(o, out);
    });
}

int ref_merge_pool_bwd(int64_t n, int64_t dim, int64_t r, int k_m, const int64_t* retained,
                       const int64_t* pool_idx, const double* pool_dist, const int32_t* pool_cnt,
                       const double* feats, const double* scores, double p, int prec,
                       const double* dout, double* dfeats, double* dscores, double* dp) {
    return guarded([&] {
        auto op = make_merge_pool_op(plan_from(r, k_m, retained, pool_idx, pool_dist, pool_cnt));
        Precision pr = prec_of(prec);
        Tensor f = from(feats, {n, dim}, pr);
        Tensor s = from(scores, {n, 1}, pr);
        Tensor pt = Tensor::full({1, 1}, p, pr);
        Tensor g = from(dout, {r, 2 * dim}, pr);
        Tensor df = Tensor::zeros({n, dim}, Precision::b64);
        Tensor ds = Tensor::zeros({n, 1}, Precision::b64);
        Tensor dpt = Tensor::zeros({1, 1}, Precision::b64);
        op->backward(g, {&f, &s, &pt}, {&df, &ds, &dpt});
        to(df, dfeats);
        to(ds, dscores);
        *dp = dpt.get(0);
    });
}

// importance_scores (merging.cpp:31-48): feats [n, d], w1 [d, h], b1 [h], w2 [h], b2
int ref_importance_scores(const double* feats, int64_t n, int64_t d, const double* w1, const double* b1,
                          const double* w2, double b2, int h, int prec, double* out) {
    return guarded([&] {
        MergeParams mp;
        mp.scorer_w1 = from(w1, {d, h}, Precision::b32);
        mp.scorer_b1 = from(b1, {1, h}, Precision::b32);
        mp.scorer_w2 = from(w2, {h, 1}, Precision::b32);
        mp.scorer_b2 = Tensor::full({1, 1}, b2, Precision::b32);
        Tensor f = from(feats, {n, d}, prec_of(prec));
        to(importance_scores(f, mp), out);
    });
}

// merge_tokens (merging.cpp:242-273): coords [n, 2], feats [n, d], scores [n], retained [r]
// ascending, proj_w [2d, d], gamma / beta [d] -> merged feats [r, d], coords [r, 2]
int ref_merge_tokens(const float* coords, const double* feats, int64_t n, int64_t d, const double* scores,
                     const int64_t* retained, int64_t r, int k_m, double p, const double* proj_w,
                     const double* gamma, const double* beta, int prec, double* out_feats, double* out_coords) {
    return guarded([&] {
        PointSet ps = points(coords, n);
        ps.feats = from(feats, {n, d}, prec_of(prec));
        Tensor s = from(scores, {n, 1}, prec_of(prec));
        MergeParams mp;
        mp.k_m = k_m;
        mp.p_merge = Tensor::full({1, 1}, p, prec_of(prec));
        mp.proj_w = from(proj_w, {2 * d, d}, prec_of(prec));
        mp.ln_gamma = from(gamma, {1, d}, prec_of(prec));
        mp.ln_beta = from(beta, {1, d}, prec_of(prec));
        MergeResult res = merge_tokens(ps, s, std::span<const int64_t>(retained, size_t(r)), mp);
        to(res.points.feats, out_feats);
        to(res.points.coords, out_coords);
    });
}

// make_interp_op (interpolation.hpp:60) forward / backward: queries [nq,2],
// key coords [nk,2], feats [nk,dim], neighbour rows idx/valid [nq,k]
int ref_interp_fwd(int64_t nq, int64_t nk, int64_t dim, int64_t k, const double* queries,
                   const float* key_coords, const double* feats, const int64_t* idx, const uint8_t* valid,
                   double p, double eps, int prec, double* out) {
    return guarded([&] {
        Precision pr = prec_of(prec);
        auto op = make_interp_op(from_f(key_coords, {nk, 2}, Precision::b64), nbr_from(idx, valid, nq, k), eps);
        Tensor f = from(feats, {nk, dim}, pr);
        Tensor pt = Tensor::full({1, 1}, p, pr);
        Tensor q = from(queries, {nq, 2}, pr);
        to(op->forward({&f, &pt, &q}), out);
    });
}

int ref_interp_bwd(int64_t nq, int64_t nk, int64_t dim, int64_t k, const double* queries,
                   const float* key_coords, const double* feats, const int64_t* idx, const uint8_t* valid,
                   double p, double eps, int prec, const double* dout, double* dfeats, double* dp,
                   double* dq) {
    return guarded([&] {
        Precision pr = prec_of(prec);
        auto op = make_interp_op(from_f(key_coords, {nk, 2}, Precision::b64), nbr_from(idx, valid, nq, k), eps);
        Tensor f = from(feats, {nk, dim}, pr);
        Tensor pt = Tensor::full({1, 1}, p, pr);
        Tensor q = from(queries, {nq, 2}, pr);
        Tensor g = from(dout, {nq, dim}, pr);
        Tensor df = Tensor::zeros({nk, dim}, Precision::b64);
        Tensor dpt = Tensor::zeros({1, 1}, Precision::b64);
        Tensor dqt = Tensor::zeros({nq, 2}, Precision::b64);
        op->backward(g, {&f, &pt, &q}, {&df, &dpt, &dqt});
        to(df, dfeats);
        *dp = dpt.get(0);
        to(dqt, dq);
    });
}

// AdamW (pipeline.cpp:639-680): `steps` optimizer steps over n_params tensors of
// rows[i] x cols[i] (b32 values, decay iff rows > 1), grads [steps][P] in tensor
// order; values [P] in, updated in place.
int ref_adamw(double lr, int64_t warmup, double wd, double beta1, double beta2, int64_t total, int64_t n_params,
              const int64_t* rows, const int64_t* cols, int64_t steps, const double* grads, double* values) {
    return guarded([&] {
        OptimConfig oc;
        oc.lr = lr;
        oc.warmup = warmup;
        oc.weight_decay = wd;
        oc.beta1 = beta1;
        oc.beta2 = beta2;
        AdamW opt(oc, total);
        std::vector<Parameter> ps;
        int64_t total_el = 0;
        for (int64_t i = 0; i < n_params; ++i) {
            Tensor v = from(values + total_el, {rows[i], cols[i]}, Precision::b32);
            ps.emplace_back("p" + std::to_string(i), v);
            total_el += rows[i] * cols[i];
        }
        std::vector<Parameter*> pp;
        for (auto& q : ps) pp.push_back(&q);
        for (int64_t st = 0; st < steps; ++st) {
            int64_t o = 0;
            for (auto& q : ps) {
                for (int64_t e = 0; e < q.value.numel(); ++e) q.grad.set(e, grads[st * total_el + o + e]);
                o += q.value.numel();
            }
            opt.step(pp);
        }
        int64_t o = 0;
        for (auto& q : ps) {
            for (int64_t e = 0; e < q.value.numel(); ++e) values[o + e] = q.value.get(e);
            o += q.value.numel();
        }
    });
}

int ref_synth_image(int64_t size, uint64_t seed, double* out) {
    return guarded([&] {
        Tensor t = synth_image(size, seed);
        for (int64_t i = 0; i < t.numel(); ++i) out[i] = t.get(i);
    });
}

int ref_write_aft(const char* path, const double* vals, const int64_t* dims, int ndim, int prec) {
    return guarded([&] {
        Tensor t = Tensor::zeros(std::vector<int64_t>(dims, dims + ndim), Precision(prec));
        for (int64_t i = 0; i < t.numel(); ++i) t.set(i, vals[i]);
        write_aft(path, t);
    });
}

int ref_write_aft_u8(const char* path, const uint8_t* bytes, const int64_t* dims, int ndim) {
    return guarded([&] {
        std::vector<int64_t> d(dims, dims + ndim);
        int64_t n = 1;
        for (int64_t x : d) n *= x;
        write_aft_u8(path, d, std::vector<uint8_t>(bytes, bytes + n));
    });
}

int ref_read_aft(const char* path, double* out, int64_t cap, int64_t* numel, int* dtype) {
    return guarded([&] {
        uint8_t dt = 0;
        Tensor t = read_aft(path, &dt);
        if (t.numel() > cap) throw ConfigError("ref_read_aft: capacity");
        for (int64_t i = 0; i < t.numel(); ++i) out[i] = t.get(i);
        *numel = t.numel();
        *dtype = dt;
    });
}

// load_checkpoint (proj/src/pipeline.cpp:772-797) into a ParamStore of `n` parameters
// named names[i] with numels[i] elements (1 x numel b32 tensors); values concatenated
// into out.  Checks that a directory written by our side loads in the reference.
int ref_load_checkpoint(const char* dir, int n, const char* const* names, const int64_t* numels,
                        double* out) {
    return guarded([&] {
        ParamStore store;
        for (int i = 0; i < n; ++i) store.add(names[i], Tensor::zeros({1, numels[i]}, Precision::b32));
        load_checkpoint(dir, store);
        int64_t o = 0;
        for (int i = 0; i < n; ++i) {
            const Tensor& v = store.find(names[i])->value;
            for (int64_t e = 0; e < v.numel(); ++e) out[o + e] = v.get(e);
            o += v.numel();
        }
    });
}

// ---- the reference Model (proj/src/pipeline.cpp) for the training-step parity tests.
// Mirrors affmae_model_cfg (include/affmae_b200.h) field for field (plain C layout).
struct RefStageCfg {
    int64_t dim;
    int heads;
    int blocks;
    int64_t cluster;
    int groups;
    double d_s;
    int interp_k;
};
struct RefAdamCfg {
    double lr;
    int64_t warmup;
    double weight_decay, beta1, beta2;
    int64_t total_steps;
};
struct RefModelCfg {
    int64_t image, patch;
    int n_stages;
    RefStageCfg stages[8];
    int64_t dec_dim;
    int dec_depth, dec_heads, gather_k, self_k;
    double lambda_aux;
    int mask_strategy;
    double mask_ratio;
    RefAdamCfg optim;
    uint64_t seed;
    int bias_hidden, scorer_hidden, merge_k;
    int64_t batch;
};

static PipelineConfig to_pipeline(const RefModelCfg& c) {
    PipelineConfig p;
    p.image = c.image;
    p.patch = c.patch;
    for (int s = 0; s < c.n_stages; ++s) {
        StageConfig st;
        st.dim = c.stages[s].dim;
        st.heads = c.stages[s].heads;
        st.blocks = c.stages[s].blocks;
        st.cluster = c.stages[s].cluster;
        st.groups = c.stages[s].groups;
        st.d_s = c.stages[s].d_s;
        st.interp_k = c.stages[s].interp_k;
        p.stages.push_back(st);
    }
    p.decoder.dim = c.dec_dim;
    p.decoder.depth = c.dec_depth;
    p.decoder.heads = c.dec_heads;
    p.decoder.gather_k = c.gather_k;
    p.decoder.self_k = c.self_k;
    p.lambda_aux = c.lambda_aux;
    p.mask_strategy = c.mask_strategy == 0 ? "perlin" : "random";
    p.mask_ratio = c.mask_ratio;
    p.optim.lr = c.optim.lr;
    p.optim.warmup = c.optim.warmup;
    p.optim.weight_decay = c.optim.weight_decay;
    p.optim.beta1 = c.optim.beta1;
    p.optim.beta2 = c.optim.beta2;
    p.seed = c.seed;
    p.bias_hidden = c.bias_hidden;
    p.scorer_hidden = c.scorer_hidden;
    p.merge_k = c.merge_k;
    return p;
}

void* ref_model_create(const RefModelCfg* cfg) {
    Model* m = nullptr;
    int rc = guarded([&] { m = new Model(to_pipeline(*cfg)); });
    return rc ? nullptr : m;
}
void ref_model_destroy(void* h) { delete static_cast<Model*>(h); }
int ref_model_param_count(void* h) { return int(static_cast<Model*>(h)->params().size()); }
const char* ref_model_param_name(void* h, int i) { return static_cast<Model*>(h)->params().all()[size_t(i)]->name.c_str(); }
int64_t ref_model_param_numel(void* h, int i) { return static_cast<Model*>(h)->params().all()[size_t(i)]->value.numel(); }
int ref_model_get(void* h, int which, double* out) {  // 0 values, 1 grads
    return guarded([&] {
        int64_t o = 0;
        for (Parameter* p : static_cast<Model*>(h)->params().all()) {
            const Tensor& t = which ? p->grad : p->value;
            for (int64_t i = 0; i < p->value.numel(); ++i) out[o + i] = which && t.numel() == 0 ? 0.0 : t.get(i);
            o += p->value.numel();
        }
    });
}
int ref_model_set(void* h, const double* in) {
    return guarded([&] {
        int64_t o = 0;
        for (Parameter* p : static_cast<Model*>(h)->params().all()) {
            for (int64_t i = 0; i < p->value.numel(); ++i) p->value.set(i, in[o + i]);
            o += p->value.numel();
        }
    });
}

// One image: encode + decode + deep_sup + loss_parts + backward (the body of train(),
// pipeline.cpp:702-727, without the optimizer).  image [S*S] (b64 like synth_image),
// masked [g*g] (1 = hidden).  loss3 = {total, main, aux}; coords_out receives every
// stage's entering coordinates concatenated (N_s x 2 each).
int ref_model_fwd_bwd(void* h, const double* image, int64_t size, const uint8_t* masked, double* loss3,
                      float* coords_out, double* feats_out) {
    return guarded([&] {
        Model& m = *static_cast<Model*>(h);
        Tensor img = Tensor::zeros({size, size}, Precision::b64);
        for (int64_t i = 0; i < img.numel(); ++i) img.set(i, image[i]);
        MaskSpec mask;
        mask.hp = mask.wp = size / m.config().patch;
        mask.patch = m.config().patch;
        mask.ratio = m.config().mask_ratio;
        mask.masked.assign(masked, masked + mask.hp * mask.wp);
        Tape t(m.precision());
        EncodeResult enc = m.encode(t, img, mask);
        int recon = m.decode(t, enc, mask);
        std::vector<int> aux;
        if (m.config().lambda_aux > 0.0) aux = m.deep_sup(t, enc, mask);
        Model::LossNodes ln = m.loss_parts(t, recon, aux, img, mask);
        loss3[0] = t.value(ln.total).get(0);
        loss3[1] = ln.main >= 0 ? t.value(ln.main).get(0) : 0.0;
        loss3[2] = ln.aux >= 0 ? t.value(ln.aux).get(0) : 0.0;
        int64_t o = 0;
        for (const EncodeStage& st : enc.stages)
            for (int64_t i = 0; i < st.coords.numel(); ++i) coords_out[o++] = float(st.coords.get(i));
        if (feats_out) {
            o = 0;
            for (const EncodeStage& st : enc.stages) {
                const Tensor& f = t.value(st.feats);
                for (int64_t i = 0; i < f.numel(); ++i) feats_out[o++] = f.get(i);
            }
        }
        m.params().zero_grads();
        t.backward(ln.total);
    });
}

// train() (pipeline.cpp:682-746) for `steps` steps over `n_images` images; losses [steps]
int ref_model_train(void* h, int64_t steps, int64_t n_images, const double* images, int64_t size, double* losses) {
    return guarded([&] {
        Model& m = *static_cast<Model*>(h);
        std::vector<Tensor> imgs;
        for (int64_t k = 0; k < n_images; ++k) {
            Tensor t = Tensor::zeros({size, size}, Precision::b64);
            for (int64_t i = 0; i < t.numel(); ++i) t.set(i, images[k * size * size + i]);
            imgs.push_back(std::move(t));
        }
        TrainResult r = train(m, steps, imgs);
        for (int64_t s = 0; s < steps; ++s) losses[s] = r.log[size_t(s)].loss;
    });
}

// mask of Model::make_mask(seed) (pipeline.cpp:625-637)
int ref_model_make_mask(void* h, uint64_t seed, uint8_t* masked) {
    return guarded([&] {
        MaskSpec ms = static_cast<Model*>(h)->make_mask(seed);
        std::memcpy(masked, ms.masked.data(), ms.masked.size());
    });
}

// Multi-core CPU baseline of the pretraining step: `threads` std::threads, each with its own
// Model replica (Parameter::grad is single-writer), each running train() over
// its share of `images` one-step images; returns the images processed.
int ref_model_train_threads(const RefModelCfg* cfg, int threads, int64_t images_per_thread, const double* image,
                            int64_t size, double* checksum) {
    return guarded([&] {
        std::vector<std::thread> pool;
        std::vector<double> sums(size_t(threads), 0.0);
        std::atomic<int> err{0};
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    Model m(to_pipeline(*cfg));
                    Tensor img = Tensor::zeros({size, size}, Precision::b64);
                    for (int64_t i = 0; i < img.numel(); ++i) img.set(i, image[i]);
                    TrainResult r = train(m, images_per_thread, {img});
                    sums[size_t(t)] = r.last_loss;
                } catch (...) {
                    err = 1;
                }
            });
        for (auto& th : pool) th.join();
        if (err) throw std::runtime_error("ref_model_train_threads: a worker failed");
        double s = 0;
        for (double v : sums) s += v;
        *checksum = s;
    });
}

// masked [grid*grid] (1 = hidden) from perlin_field(grid, grid, 2, 4.0, 0.5, seed)
int ref_perlin_mask(int64_t grid, double ratio, uint64_t seed, uint8_t* masked) {
    return guarded([&] {
        MaskSpec m = mask_from_field(perlin_field(grid, grid, kPerlinOctaves, kPerlinBaseFreq,
                                                  kPerlinPersistence, seed),
                                     ratio);
        std::memcpy(masked, m.masked.data(), m.masked.size());
    });
}

// The multi-core CPU baseline: for each of `images` images, on `threads`
// std::threads, run the reference hot path exactly as Model::encode wires it
// (proj/src/pipeline.cpp:436-465) for one attention layer: balanced_clusters
// -> cluster_neighborhood -> nbhd_attn_streaming -> nbhd_attn_backward ->
// select_retained -> merge_plan -> merge pool forward + backward.  Inputs are
// per image: coords [n,2], q/k/v/dout [n,hd], scores [n], feats [n,hd];
// shared: blanks [h,d], bias params, p.  `stages` selects what runs
// (bit 0 index, 1 attn fwd, 2 attn bwd, 3 merge).  Returns a checksum of the
// outputs in *checksum so the work cannot be elided.
int ref_hotpath_batch(int64_t images, int threads, int stages, int64_t n, int heads, int d,
                      int hidden, double patch, int64_t cluster, int64_t groups, double d_s,
                      int k_m, const float* coords, const double* q, const double* k,
                      const double* v, const double* dout, const double* scores,
                      const double* bk, const double* bv, const double* w1, const double* b1,
                      const double* w2, const double* b2, const double* blank, double p,
                      double* checksum) {
    return guarded([&] {
        int64_t hd = int64_t(heads) * d;
        std::vector<double> sums(size_t(images), 0.0);
        std::atomic<int64_t> next{0};
        std::vector<std::string> errs(static_cast<size_t>(threads), std::string());
        auto worker = [&](int tid) {
            try {
                for (;;) {
                    int64_t b = next.fetch_add(1);
                    if (b >= images) break;
                    double acc = 0.0;
                    PointSet ps = points(coords + b * n * 2, n);
                    ClusterAssignment a = balanced_clusters(ps, cluster);
                    NeighborIndex nb = cluster_neighborhood(a, ps, groups);
                    acc += double(nb.width);
                    if (stages & 6) {
                        AttnInputs in;
                        in.q = from(q + b * n * hd, {n, hd}, Precision::b32);
                        in.k = from(k + b * n * hd, {n, hd}, Precision::b32);
                        in.v = from(v + b * n * hd, {n, hd}, Precision::b32);
                        in.bk = from(bk, {heads, d}, Precision::b32);
                        in.bv = from(bv, {heads, d}, Precision::b32);
                        in.coords = ps.coords;
                        in.nbr = nb;
                        in.bias.heads = heads;
                        in.bias.hidden = hidden;
                        in.bias.patch = patch;
                        in.bias.w1 = from(w1, {heads, 2 * hidden}, Precision::b32);
                        in.bias.b1 = from(b1, {heads, hidden}, Precision::b32);
                        in.bias.w2 = from(w2, {heads, hidden}, Precision::b32);
                        in.bias.b2 = from(b2, {heads, 1}, Precision::b32);
                        in.bias.blank = from(blank, {heads, 1}, Precision::b32);
                        AttnCtx c = in.ctx(heads, d);
                        if (stages & 2) acc += nbhd_attn_streaming(c).get(0);
                        if (stages & 4) {
                            Tensor cot = from(dout + b * n * hd, {n, hd}, Precision::b32);
                            acc += nbhd_attn_backward(c, cot).dq.get(0);
                        }
                    }
                    if (stages & 8) {
                        Tensor sc = from(scores + b * n, {n, 1}, Precision::b32);
                        std::vector<int64_t> ret = select_retained(sc, d_s);
                        MergePlan plan = merge_plan(ps, ret, k_m);
                        auto op = make_merge_pool_op(plan);
                        Tensor f = from(q + b * n * hd, {n, hd}, Precision::b32);
                        Tensor pt = Tensor::full({1, 1}, p, Precision::b32);
                        Tensor o = op->forward({&f, &sc, &pt});
                        Tensor df = Tensor::zeros({n, hd}, Precision::b32);
                        Tensor ds = Tensor::zeros({n, 1}, Precision::b32);
                        Tensor dpt = Tensor::zeros({1, 1}, Precision::b32);
                        op->backward(o, {&f, &sc, &pt}, {&df, &ds, &dpt});
                        acc += o.get(0) + dpt.get(0);
                    }
                    sums[size_t(b)] = acc;
                }
            } catch (const std::exception& e) {
                errs[size_t(tid)] = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t);
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        double s = 0.0;
        for (double x : sums) s += x;
        *checksum = s;
    });
}

} // extern "C"
