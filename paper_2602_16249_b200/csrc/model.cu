// Device-resident training step of the AFFMAE model (SURVEY.md §8(a) Model::encode stage
// loop, §8(f) #1-#3, BASELINE configs[2]): Model::encode / decode / deep_sup / loss_parts
// (proj/src/pipeline.cpp:402-610), the reverse sweep the reference's Tape runs over them
// (proj/src/tape.cpp:466-724) written out explicitly, and AdamW (pipeline.cpp:639-680).
//
// Everything runs on this library's kernels on one CUDA stream: the cluster index, attention
// plan / fwd / bwd, selection, merge plan / pool, knn, interpolation and decoder attention, the
// tcgen05 GEMMs, and the row kernels of model_kernels.cu.  Layout:
//   * parameters: one fp32 arena (the reference's b32 values), ParamStore order of
//     Model::Model (pipeline.cpp:255-371) except that the GEMM-operand tensors come first;
//     matrices used by a GEMM are stored transposed ([out, in], the tensor-core B operand)
//     and shadowed in bf16 (refreshed by the optimizer pass); gradients, AdamW moments the
//     same layout;
//   * activations: [B * N_s, D] rows (B images of equal token counts), bf16
//     operands and an fp32 residual stream, every tensor the backward needs kept;
//   * batched semantics: the loss is the mean over images of the reference's per-image
//     loss, so B = 1 reproduces the reference's step.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "model_kernels.h"

namespace affmae_b200 {
namespace {

using bf16 = __nv_bfloat16;

// --------------------------------------------------------------- host RNG
// splitmix64 + Box-Muller exactly as proj/include/affmae/rng.hpp:8-55 (the parameter init
// and the random mask strategy draw from it).
uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double normal() {
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
    uint64_t below(uint64_t n) { return n ? next() % n : 0; }
};

constexpr int kPosHidden = 16;  // pipeline.cpp:25
constexpr double kInterpEps = 1e-6;

struct Arena {
    uint8_t* base = nullptr;
    size_t off = 0;
    template <class T>
    T* take(int64_t n) {
        const size_t b = (size_t(n > 0 ? n : 1) * sizeof(T) + 255) & ~size_t(255);
        T* r = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += b;
        return r;
    }
};

struct Param {
    std::string name;
    int64_t r, c;          // reference dims
    bool tr;               // stored transposed [c][r]
    bool shadow;           // bf16 shadow (GEMM operand / attention blank rows)
    bool decay;            // dim(0) > 1 (pipeline.cpp:666)
    int kind;              // init: 0 normal(scale), 1 zeros, 2 ones
    double scale;
    int64_t off = 0;       // arena offset (floats)
    std::vector<float> init;
};

struct Blk {
    bf16 *h1, *qkv, *a, *h2, *pre, *m;  // qkv: [M, 3D] rows q | k | v (one GEMM, attention reads strided)
    float2 *st1, *st2;
    float* lse;
    float* fmid;
};

struct Stage {
    int64_t N, D, M, R = 0;
    int heads;
    affmae_cluster_geom geom;
    affmae_attn_desc desc;
    float* coords;
    affmae_cluster_index idx;
    affmae_attn_plan plan;
    std::vector<float*> f;  // blocks + 1 residual buffers
    std::vector<Blk> blk;
    bf16* fout_bf;
    float* df;  // gradient of f[blocks] (-> of f[0] after the blocks' backward)
    // merge (all stages but the last)
    bf16 *shid = nullptr, *spre = nullptr, *pooled = nullptr, *ymerge = nullptr, *ylnm = nullptr;
    float* scores = nullptr;
    int32_t* ret = nullptr;
    int32_t* forced_ret = nullptr;  // affmae_model_force_retained (parity tests' teacher forcing)
    bool forced = false;
    affmae_merge_plan mplan{};
    float2* stm = nullptr;
    // deep supervision head (all stages but the last)
    int32_t* aidx = nullptr;
    uint8_t* aval = nullptr;
    bf16 *avirt = nullptr, *aout = nullptr, *daux = nullptr;
};

struct DecRound {
    float *fq_in, *fq_x, *fq_s, *fq_out;
    float *offpre, *qpos;
    int32_t* gidx;
    uint8_t* gval;
    bf16* virt;
    // q1 [M, dd]; kv1 [M, 2dd] = k1 | v1 (one GEMM from the virtual tokens); qkv2 [M, 3dd]
    // = q2 | k2 | v2 (one GEMM from h2): the attention kernels read them as strided slices
    bf16 *h1, *q1, *kv1, *a1, *h2, *qkv2, *a2, *h3, *pre, *m;
    float *lse1, *lse2;
    float2 *st1, *st2, *st3;
};

struct DecStage {
    bf16 *hz, *zpos, *z;
    std::vector<DecRound> rounds;
};

__global__ void loss_combine_kernel(float* loss, int n_aux, float lambda) {
    // loss: [0] total, [1] main, [2] aux mean, [3..] per-stage aux terms (Model::loss_parts)
    float s = 0.f;
    for (int i = 0; i < n_aux; ++i) s += loss[3 + i];
    const float aux = n_aux ? s / float(n_aux) : 0.f;
    loss[2] = aux;
    loss[0] = loss[1] + (n_aux ? lambda * aux : 0.f);
}

__global__ void fill_one_to_one_kernel(int32_t* idx, uint8_t* val, int64_t batch, int64_t q) {
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < batch * q; t += int64_t(gridDim.x) * blockDim.x) {
        idx[t] = int32_t(t % q);
        val[t] = 1;
    }
}

}  // namespace
}  // namespace affmae_b200

// The opaque handle of the C ABI.
struct affmae_model {
    affmae_model_cfg cfg{};
    int ns = 0;
    int64_t B = 0, S = 0, g = 0, cells = 0, p2 = 0, Q = 0, Mq = 0, dd = 0;
    std::vector<int64_t> N;
    std::vector<affmae_b200::Param> params;
    std::map<std::string, int> pidx;
    int64_t nvals = 0, nshadow = 0;

    uint8_t* dmem = nullptr;
    size_t dbytes = 0;
    float *P = nullptr, *G = nullptr, *M1 = nullptr, *V1 = nullptr;
    __nv_bfloat16* PB = nullptr;
    int64_t* seg_off = nullptr;
    uint8_t* seg_decay = nullptr;
    int64_t* step_dev = nullptr;
    void* adam_scalars = nullptr;
    float* zero_bias = nullptr;

    double* images = nullptr;
    uint8_t* masked = nullptr;
    float* patches = nullptr;
    int32_t *vis_rows = nullptr, *msk_rows = nullptr;
    __nv_bfloat16 *vec = nullptr, *h0 = nullptr, *ypos0 = nullptr, *emb = nullptr;
    std::vector<affmae_b200::Stage> st;

    float* refs = nullptr;
    int32_t *self_idx = nullptr, *one_idx = nullptr;
    uint8_t *self_val = nullptr, *one_val = nullptr;
    __nv_bfloat16 *hq = nullptr, *yposq = nullptr, *hh = nullptr, *recon = nullptr, *drecon = nullptr;
    float *fq0 = nullptr, *fq_final = nullptr;
    float2* sth = nullptr;
    std::vector<affmae_b200::DecStage> dec;
    float* loss = nullptr;

    // scratch
    uint8_t* ws = nullptr;
    size_t ws_bytes = 0;
    uint8_t* gws = nullptr;
    size_t gws_bytes = 0;
    float* part = nullptr;
    float *F1 = nullptr, *F2 = nullptr, *F3 = nullptr, *F4 = nullptr, *F5 = nullptr, *dz = nullptr, *dscores = nullptr;
    float *dfq = nullptr, *dqpos = nullptr, *dqjunk = nullptr;
    __nv_bfloat16 *T1 = nullptr, *B1 = nullptr, *B2 = nullptr, *B4 = nullptr,
                  *B6 = nullptr, *dfbf = nullptr, *dfq_bf = nullptr;
    // second copies of the scratch the side-stream weight gradients read, so the main stream's
    // next writer does not have to wait for them (see Ctx::side_dw)
    __nv_bfloat16 *B4b = nullptr, *dfbf2 = nullptr, *dfq_bf2 = nullptr, *B2x = nullptr;
    // decoder: dY of the fused self-attention q | k | v and cross-attention k | v projections
    __nv_bfloat16 *dqkv = nullptr, *dkv = nullptr;
    cudaStream_t side = nullptr;       // weight-gradient GEMMs of the backward
    std::vector<cudaEvent_t> events;   // fork / join events of one step (reused every step)
    uint8_t* gws2 = nullptr;           // GEMM workspace of the side stream

    int64_t steps = 0;
    int world = 1;          // data-parallel ranks: the loss gradient is seeded with 1/world
    void* comm = nullptr;   // NCCL communicator (dist.cu) or null (single GPU / caller reduces)
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t gstream = nullptr;
    float* gloss = nullptr;
};

namespace affmae_b200 {
namespace {

using Model = affmae_model;

#define CK(expr)                      \
    do {                              \
        int _rc = (expr);             \
        if (_rc) return _rc;          \
    } while (0)

int64_t round8(int64_t x) { return (x + 7) / 8 * 8; }

// ------------------------------------------------------------ parameter table
// Model::Model (pipeline.cpp:255-371), in the reference's insertion order
void build_params(Model& m) {
    const affmae_model_cfg& c = m.cfg;
    auto add = [&](const std::string& n, int64_t r, int64_t cc, int kind, double scale, bool tr, bool sh) {
        Param p;
        p.name = n;
        p.r = r;
        p.c = cc;
        p.kind = kind;
        p.scale = scale;
        p.tr = tr;
        p.shadow = sh;
        p.decay = r > 1;
        m.pidx[n] = int(m.params.size());
        m.params.push_back(std::move(p));
    };
    // mat: normal / sqrt(rows); GEMM operands are transposed + shadowed
    auto mat = [&](const std::string& n, int64_t r, int64_t cc, bool gemm = true) {
        add(n, r, cc, 0, 1.0 / std::sqrt(double(r)), true, gemm);
    };
    auto small = [&](const std::string& n, int64_t r, int64_t cc, bool sh) { add(n, r, cc, 0, 0.02, false, sh); };
    auto zero = [&](const std::string& n, int64_t r, int64_t cc) { add(n, r, cc, 1, 0.0, false, false); };
    auto one = [&](const std::string& n, int64_t cc) { add(n, 1, cc, 2, 0.0, false, false); };
    auto full1 = [&](const std::string& n) { add(n, 1, 1, 2, 0.0, false, false); };
    auto pos_net = [&](const std::string& pre, int64_t out) {
        mat(pre + ".w1", 2, kPosHidden, false);  // custom kernel reads it as [16][2]
        zero(pre + ".b1", 1, kPosHidden);
        mat(pre + ".w2", kPosHidden, out);
        zero(pre + ".b2", 1, out);
    };
    auto bias_net = [&](const std::string& pre, int64_t heads) {
        const int64_t hb = c.bias_hidden;
        add(pre + ".w1", heads, 2 * hb, 0, 1.0 / std::sqrt(2.0), false, false);
        zero(pre + ".b1", heads, hb);
        add(pre + ".w2", heads, hb, 0, 1.0 / std::sqrt(double(hb)), false, false);
        zero(pre + ".b2", heads, 1);
        zero(pre + ".blank", heads, 1);
    };
    auto attn_block = [&](const std::string& pre, int64_t dim, int heads) {
        mat(pre + "wq", dim, dim);
        mat(pre + "wk", dim, dim);
        mat(pre + "wv", dim, dim);
        mat(pre + "wo", dim, dim);
        small(pre + "blank_k", heads, dim / heads, true);
        small(pre + "blank_v", heads, dim / heads, true);
        bias_net(pre + "bias", heads);
    };
    const int64_t p2 = c.patch * c.patch, d0 = c.stages[0].dim;
    mat("embed.w", p2, d0);
    zero("embed.b", 1, d0);
    pos_net("pos0", d0);
    for (int s = 0; s < c.n_stages; ++s) {
        const affmae_stage_cfg& sc = c.stages[s];
        for (int b = 0; b < sc.blocks; ++b) {
            const std::string pre = "enc.s" + std::to_string(s) + ".b" + std::to_string(b) + ".";
            one(pre + "ln1.g", sc.dim);
            zero(pre + "ln1.b", 1, sc.dim);
            attn_block(pre, sc.dim, sc.heads);
            one(pre + "ln2.g", sc.dim);
            zero(pre + "ln2.b", 1, sc.dim);
            mat(pre + "mlp.w1", sc.dim, 4 * sc.dim);
            zero(pre + "mlp.b1", 1, 4 * sc.dim);
            mat(pre + "mlp.w2", 4 * sc.dim, sc.dim);
            zero(pre + "mlp.b2", 1, sc.dim);
        }
        if (s + 1 < c.n_stages) {
            const int64_t dn = c.stages[s + 1].dim;
            const std::string pre = "merge.s" + std::to_string(s) + ".";
            mat(pre + "scorer.w1", sc.dim, c.scorer_hidden);
            zero(pre + "scorer.b1", 1, c.scorer_hidden);
            mat(pre + "scorer.w2", c.scorer_hidden, 1, false);  // [1][16]: the output unit's weights
            zero(pre + "scorer.b2", 1, 1);
            full1(pre + "p");
            mat(pre + "proj", 2 * sc.dim, dn);
            one(pre + "ln.g", dn);
            zero(pre + "ln.b", 1, dn);
        }
    }
    const int64_t dd = c.dec_dim;
    const int hd = c.dec_heads;
    small("dec.mask_token", 1, dd, false);
    pos_net("dec.pos", dd);
    for (int s = 0; s < c.n_stages; ++s) {
        const std::string sp = "dec.s" + std::to_string(s) + ".";
        mat(sp + "in.w", c.stages[s].dim, dd);
        zero(sp + "in.b", 1, dd);
        for (int r = 0; r < c.dec_depth; ++r) {
            const std::string pre = sp + "r" + std::to_string(r) + ".";
            add(pre + "off.w", dd, 2, 1, 0.0, true, false);  // zero init, read as [2][dd]
            zero(pre + "off.b", 1, 2);
            full1(pre + "p");
            one(pre + "ln1.g", dd);
            zero(pre + "ln1.b", 1, dd);
            attn_block(pre + "x.", dd, hd);
            one(pre + "ln2.g", dd);
            zero(pre + "ln2.b", 1, dd);
            attn_block(pre + "s.", dd, hd);
            one(pre + "ln3.g", dd);
            zero(pre + "ln3.b", 1, dd);
            mat(pre + "mlp.w1", dd, 2 * dd);
            zero(pre + "mlp.b1", 1, 2 * dd);
            mat(pre + "mlp.w2", 2 * dd, dd);
            zero(pre + "mlp.b2", 1, dd);
        }
    }
    one("dec.head.ln.g", dd);
    zero("dec.head.ln.b", 1, dd);
    mat("dec.head.w", dd, p2);
    zero("dec.head.b", 1, p2);
    for (int s = 0; s + 1 < c.n_stages; ++s) {
        const std::string pre = "aux.s" + std::to_string(s) + ".";
        full1(pre + "p");
        mat(pre + "w", c.stages[s].dim, p2);
        zero(pre + "b", 1, p2);
    }
    // the draws, in insertion order (normal_init, pipeline.cpp:40-45), stored as fp32
    Rng rng(mix64(c.seed ^ 0x1417ull));
    for (Param& p : m.params) {
        const int64_t n = p.r * p.c;
        p.init.assign(size_t(n), 0.f);
        if (p.kind == 2) std::fill(p.init.begin(), p.init.end(), 1.f);
        if (p.kind != 0) continue;
        for (int64_t i = 0; i < n; ++i) p.init[size_t(i)] = float(rng.normal() * p.scale);
    }
    // arena: shadowed tensors first (one contiguous bf16 shadow), each padded to 8 values
    int64_t off = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (Param& p : m.params) {
            if (p.shadow != (pass == 0)) continue;
            p.off = off;
            off += round8(p.r * p.c);
            if (pass == 0) m.nshadow = off;
        }
    m.nvals = off;
}

// reference layout <-> arena layout
void to_arena(const Param& p, const float* ref, float* arena) {
    float* dst = arena + p.off;
    if (!p.tr) {
        std::memcpy(dst, ref, sizeof(float) * size_t(p.r * p.c));
        return;
    }
    for (int64_t i = 0; i < p.r; ++i)
        for (int64_t j = 0; j < p.c; ++j) dst[j * p.r + i] = ref[i * p.c + j];
}
void from_arena(const Param& p, const float* arena, float* ref) {
    const float* src = arena + p.off;
    if (!p.tr) {
        std::memcpy(ref, src, sizeof(float) * size_t(p.r * p.c));
        return;
    }
    for (int64_t i = 0; i < p.r; ++i)
        for (int64_t j = 0; j < p.c; ++j) ref[i * p.c + j] = src[j * p.r + i];
}

float* PF(Model& m, const std::string& n) { return m.P + m.params[size_t(m.pidx.at(n))].off; }
float* GF(Model& m, const std::string& n) { return m.G + m.params[size_t(m.pidx.at(n))].off; }
bf16* PBF(Model& m, const std::string& n) { return m.PB + m.params[size_t(m.pidx.at(n))].off; }

// ------------------------------------------------------------------- layout
void layout(Model& m, Arena& a) {
    const affmae_model_cfg& c = m.cfg;
    const int64_t B = m.B, dd = m.dd, p2 = m.p2, Mq = m.Mq;
    m.P = a.take<float>(m.nvals);
    m.G = a.take<float>(m.nvals);
    m.M1 = a.take<float>(m.nvals);
    m.V1 = a.take<float>(m.nvals);
    m.PB = a.take<bf16>(m.nshadow);
    m.seg_off = a.take<int64_t>(int64_t(m.params.size()));
    m.seg_decay = a.take<uint8_t>(int64_t(m.params.size()));
    m.step_dev = a.take<int64_t>(1);
    m.adam_scalars = a.take<uint8_t>(int64_t(adamw_scalars_bytes()));
    int64_t maxn = p2;
    for (int s = 0; s < m.ns; ++s) maxn = std::max<int64_t>(maxn, 4 * c.stages[s].dim);
    maxn = std::max<int64_t>(maxn, 2 * dd);
    m.zero_bias = a.take<float>(maxn);
    m.loss = a.take<float>(8 + m.ns);

    m.images = a.take<double>(B * m.S * m.S);
    m.masked = a.take<uint8_t>(B * m.cells);
    m.patches = a.take<float>(B * m.cells * p2);
    m.vis_rows = a.take<int32_t>(B * m.N[0]);
    m.msk_rows = a.take<int32_t>(Mq);
    const int64_t M0 = B * m.N[0];
    m.vec = a.take<bf16>(round8(M0) * p2);
    m.h0 = a.take<bf16>(round8(M0) * kPosHidden);
    m.ypos0 = a.take<bf16>(round8(M0) * c.stages[0].dim);
    m.emb = a.take<bf16>(round8(M0) * c.stages[0].dim);

    for (int s = 0; s < m.ns; ++s) {
        Stage& S = m.st[size_t(s)];
        const affmae_stage_cfg& sc = c.stages[s];
        const int64_t M = S.M, D = S.D, Mp = round8(M);
        S.coords = a.take<float>(M * 2);
        S.idx.perm = a.take<int32_t>(M);
        S.idx.cluster_of = a.take<int32_t>(M);
        S.idx.nbr_cl = a.take<int32_t>(B * S.geom.n_clusters * S.geom.groups_eff);
        S.idx.rev_off = a.take<int32_t>(B * (S.geom.n_clusters + 1));
        S.idx.rev_cl = a.take<int32_t>(B * S.geom.n_clusters * S.geom.groups_eff);
        S.plan.bytes = attn_plan_workspace(&S.geom, 1);
        S.plan.buf = a.take<uint8_t>(int64_t(S.plan.bytes));
        S.f.assign(size_t(sc.blocks + 1), nullptr);
        for (auto& f : S.f) f = a.take<float>(Mp * D);
        S.blk.resize(size_t(sc.blocks));
        for (Blk& k : S.blk) {
            k.h1 = a.take<bf16>(Mp * D);
            k.qkv = a.take<bf16>(Mp * 3 * D);
            k.a = a.take<bf16>(Mp * D);
            k.h2 = a.take<bf16>(Mp * D);
            k.pre = a.take<bf16>(Mp * 4 * D);
            k.m = a.take<bf16>(Mp * 4 * D);
            k.st1 = a.take<float2>(Mp);
            k.st2 = a.take<float2>(Mp);
            k.lse = a.take<float>(M * S.heads);
            k.fmid = a.take<float>(Mp * D);
        }
        S.fout_bf = a.take<bf16>(Mp * D);
        S.df = a.take<float>(Mp * D);
        if (s + 1 < m.ns) {
            const int64_t R = S.R, Dn = c.stages[s + 1].dim, Mn = round8(B * R);
            S.shid = a.take<bf16>(Mp * 16);
            S.spre = a.take<bf16>(Mp * 16);
            S.scores = a.take<float>(M);
            S.ret = a.take<int32_t>(B * R);
            S.forced_ret = a.take<int32_t>(B * R);
            S.mplan.target = a.take<int32_t>(M);
            S.mplan.pool_idx = a.take<int32_t>(B * R * c.merge_k);
            S.mplan.pool_dist = a.take<double>(B * R * c.merge_k);
            S.mplan.pool_cnt = a.take<int32_t>(B * R);
            S.mplan.row_of = a.take<int32_t>(M);
            S.pooled = a.take<bf16>(Mn * 2 * D);
            S.ymerge = a.take<bf16>(Mn * Dn);
            S.ylnm = a.take<bf16>(Mn * Dn);
            S.stm = a.take<float2>(Mn);
            if (c.lambda_aux > 0.0) {
                const int k = c.stages[s].interp_k;
                S.aidx = a.take<int32_t>(Mq * k);
                S.aval = a.take<uint8_t>(Mq * k);
                S.avirt = a.take<bf16>(round8(Mq) * D);
                S.aout = a.take<bf16>(round8(Mq) * p2);
                S.daux = a.take<bf16>(round8(Mq) * p2);
            }
        }
    }
    const int64_t Mqp = round8(Mq);
    m.refs = a.take<float>(Mq * 2);
    m.self_idx = a.take<int32_t>(Mq * c.self_k);
    m.self_val = a.take<uint8_t>(Mq * c.self_k);
    m.one_idx = a.take<int32_t>(Mq);
    m.one_val = a.take<uint8_t>(Mq);
    m.hq = a.take<bf16>(Mqp * kPosHidden);
    m.yposq = a.take<bf16>(Mqp * dd);
    m.fq0 = a.take<float>(Mqp * dd);
    m.dec.resize(size_t(m.ns));
    float* prev = m.fq0;
    for (int si = m.ns - 1; si >= 0; --si) {
        DecStage& d = m.dec[size_t(si)];
        const int64_t Mp = round8(m.st[size_t(si)].M);
        d.hz = a.take<bf16>(Mp * kPosHidden);
        d.zpos = a.take<bf16>(Mp * dd);
        d.z = a.take<bf16>(Mp * dd);
        d.rounds.resize(size_t(c.dec_depth));
        for (DecRound& r : d.rounds) {
            r.fq_in = prev;
            r.fq_x = a.take<float>(Mqp * dd);
            r.fq_s = a.take<float>(Mqp * dd);
            r.fq_out = a.take<float>(Mqp * dd);
            prev = r.fq_out;
            r.offpre = a.take<float>(Mq * 2);
            r.qpos = a.take<float>(Mq * 2);
            r.gidx = a.take<int32_t>(Mq * c.gather_k);
            r.gval = a.take<uint8_t>(Mq * c.gather_k);
            r.virt = a.take<bf16>(Mqp * dd);
            for (bf16** b : {&r.h1, &r.q1, &r.a1, &r.h2, &r.a2, &r.h3}) *b = a.take<bf16>(Mqp * dd);
            r.kv1 = a.take<bf16>(Mqp * 2 * dd);
            r.qkv2 = a.take<bf16>(Mqp * 3 * dd);
            r.pre = a.take<bf16>(Mqp * 2 * dd);
            r.m = a.take<bf16>(Mqp * 2 * dd);
            r.lse1 = a.take<float>(Mq * c.dec_heads);
            r.lse2 = a.take<float>(Mq * c.dec_heads);
            r.st1 = a.take<float2>(Mqp);
            r.st2 = a.take<float2>(Mqp);
            r.st3 = a.take<float2>(Mqp);
        }
    }
    m.fq_final = prev;
    m.hh = a.take<bf16>(Mqp * dd);
    m.sth = a.take<float2>(Mqp);
    m.recon = a.take<bf16>(Mqp * p2);
    m.drecon = a.take<bf16>(Mqp * p2);

    // scratch, each sized for its largest use (rows rounded to 8)
    int64_t eMD = Mqp * dd, e16 = Mqp * kPosHidden, e4 = Mqp * 2 * dd, eB1 = Mqp * dd, eB6 = Mqp * dd, eRows = Mqp,
            eZ = 0, eDf = 0;
    for (int s = 0; s < m.ns; ++s) {
        const Stage& S = m.st[size_t(s)];
        const int64_t Mp = round8(S.M);
        eMD = std::max(eMD, Mp * S.D);
        e16 = std::max(e16, Mp * kPosHidden);
        e4 = std::max(e4, Mp * 4 * S.D);
        eB1 = std::max(eB1, std::max(Mp * S.D, Mqp * S.D));
        eB6 = std::max(eB6, Mp * dd);
        eRows = std::max(eRows, Mp);
        eZ = std::max(eZ, Mp * dd);
        eDf = std::max(eDf, Mp * S.D);
        if (s + 1 < m.ns) {
            const int64_t Mn = round8(m.B * S.R);
            eB1 = std::max(eB1, Mn * m.st[size_t(s + 1)].D);
            e4 = std::max(e4, Mn * 2 * S.D);
        }
    }
    m.F1 = a.take<float>(eMD);
    m.F2 = a.take<float>(Mqp * dd);
    m.F3 = a.take<float>(Mqp * dd);
    m.F4 = a.take<float>(Mqp * dd);
    m.F5 = a.take<float>(e16);
    m.dz = a.take<float>(eZ);
    m.dscores = a.take<float>(eRows);
    m.dfq = a.take<float>(Mqp * dd);
    m.dqpos = a.take<float>(Mq * 2);
    m.dqjunk = a.take<float>(Mq * 2);
    m.T1 = a.take<bf16>(eMD);
    m.B1 = a.take<bf16>(eB1);
    m.B2 = a.take<bf16>(e16);
    m.B4 = a.take<bf16>(e4);
    m.B6 = a.take<bf16>(eB6);
    m.dfbf = a.take<bf16>(eDf);
    m.dfbf2 = a.take<bf16>(eDf);
    m.B4b = a.take<bf16>(e4);
    m.dfq_bf2 = a.take<bf16>(Mqp * dd);
    m.B2x = a.take<bf16>(Mqp * dd);
    m.dqkv = a.take<bf16>(Mqp * 3 * dd);
    m.dkv = a.take<bf16>(Mqp * 2 * dd);
    m.dfq_bf = a.take<bf16>(Mqp * dd);
}

// ------------------------------------------------------------------ sizing
size_t part_floats(const Model& m) {
    size_t p = 0;
    auto upd = [&](size_t x) { p = std::max(p, x); };
    for (const Stage& S : m.st) {
        upd(mk::ln_bwd_part_floats(S.M, S.D));
        upd(mk::pos_part_floats(S.M));
        upd(mk::pos_part_floats(S.M) / 48 * 17 + 17);
        upd(mk::colsum_part_floats(S.D));
        if (S.R) upd(mk::ln_bwd_part_floats(m.B * S.R, m.cfg.stages[&S - &m.st[0] + 1].dim));
    }
    upd(mk::ln_bwd_part_floats(m.Mq, m.dd));
    upd(mk::offset_part_floats(m.Mq, m.dd));
    upd(mk::pos_part_floats(m.Mq));
    upd(mk::colsum_part_floats(m.dd));
    return p;
}

size_t misc_ws_bytes(const Model& m) {
    size_t w = masked_mse_workspace(m.Mq);
    auto upd = [&](size_t x) { w = std::max(w, x); };
    const affmae_model_cfg& c = m.cfg;
    for (int s = 0; s < m.ns; ++s) {
        const Stage& S = m.st[size_t(s)];
        upd(cluster_index_workspace(&S.geom));
        upd(attn_fwd_planned_workspace(&S.geom, &S.desc));
        upd(attn_bwd_planned_workspace(&S.geom, &S.desc));
        if (s + 1 < m.ns) {
            upd(select_retained_workspace(m.B, S.N));
            upd(merge_plan_workspace(m.B, S.N, S.R));
            upd(merge_pool_bwd_workspace(m.B, S.R));
        }
    }
    upd(perlin_mask_workspace(m.B, m.g, m.g, 2, 4.0));
    {
        affmae_attn_desc dd{c.dec_heads, int(m.dd / c.dec_heads), c.bias_hidden, double(c.patch)};
        upd(gattn_bwd_workspace(&dd, m.B, m.Q, c.self_k));
        // cross attention (one-to-one): per-block parameter-gradient rows
        upd(size_t(16) * device_sms() * size_t(2 * m.dd + 4 * c.dec_heads * c.bias_hidden + 2 * c.dec_heads) * 4);
    }
    for (int s = 0; s < m.ns; ++s) {
        upd(interp_bwd_gather_workspace(m.B, m.Q, m.st[size_t(s)].N, c.gather_k));
        upd(interp_bwd_gather_workspace(m.B, m.Q, m.st[size_t(s)].N, c.stages[s].interp_k));
    }
    (void)c;
    return w;
}

size_t gemm_ws_bytes(const Model& m) {
    // the tile scheduler state of the largest GEMM (+ the bias column-sum partials)
    int64_t Mmax = m.Mq, Nmax = 4 * m.dd;
    for (const Stage& S : m.st) {
        Mmax = std::max(Mmax, S.M);
        Nmax = std::max(Nmax, 4 * S.D);
    }
    size_t w = std::max(linear_workspace(round8(Mmax), Nmax, Nmax), linear_bwd_workspace(round8(Mmax), Nmax, Nmax));
    return std::max<size_t>(w, size_t(256) << 20);
}

// ------------------------------------------------------------------ GEMMs
struct Ctx {
    Model& m;
    cudaStream_t st;
    // backward only: weight gradients on m.side (off the critical dX chain); `pending` maps a
    // dY buffer to the side-stream event after its last reader, waited for before the main
    // stream overwrites it (guard)
    bool overlap = false;
    mutable std::vector<std::pair<const void*, cudaEvent_t>> pending;
    mutable size_t next_event = 0;
    void* sv() const { return reinterpret_cast<void*>(st); }
    cudaEvent_t event() const {
        if (next_event >= m.events.size()) return nullptr;
        return m.events[next_event++];
    }
    // the main stream is about to write `buf`: wait for the side-stream readers of it
    int guard(const void* buf) const {
        for (size_t i = 0; i < pending.size(); ++i)
            if (pending[i].first == buf) {
                if (cudaStreamWaitEvent(st, pending[i].second, 0) != cudaSuccess)
                    return cuda_status(cudaGetLastError(), "model guard");
                pending.erase(pending.begin() + int64_t(i));
                return AFFMAE_OK;
            }
        return AFFMAE_OK;
    }
    // dW (+db) += from x [rows, k], dy [rows, n] on the side stream (dy must stay unchanged
    // until the guard of the buffer); falls back to the main stream without overlap
    int side_dw(const bf16* x, const bf16* w, const bf16* dy, int64_t rows, int64_t n, int64_t k, float* dw,
                float* db) const {
        cudaEvent_t fork = overlap ? event() : nullptr, done = overlap ? event() : nullptr;
        if (!fork || !done) return linear_bwd(x, w, dy, rows, n, k, nullptr, dw, db, m.gws, m.gws_bytes, sv());
        if (cudaEventRecord(fork, st) != cudaSuccess || cudaStreamWaitEvent(m.side, fork, 0) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model side fork");
        CK(linear_bwd(x, w, dy, rows, n, k, nullptr, dw, db, m.gws2, m.gws_bytes, reinterpret_cast<void*>(m.side)));
        if (cudaEventRecord(done, m.side) != cudaSuccess) return cuda_status(cudaGetLastError(), "model side record");
        for (auto& pe : pending)
            if (pe.first == dy) {
                pe.second = done;  // the side stream is in order: the latest reader implies the earlier ones
                return AFFMAE_OK;
            }
        pending.emplace_back(dy, done);
        return AFFMAE_OK;
    }
    // dX = dy W (bf16) on the main stream, dW / db on the side stream
    int bwd_xw(const bf16* x, const bf16* w, const bf16* dy, int64_t rows, int64_t n, int64_t k, bf16* dx, float* dw,
               float* db) const {
        if (!overlap) return linear_bwd(x, w, dy, rows, n, k, dx, dw, db, m.gws, m.gws_bytes, sv());
        CK(side_dw(x, w, dy, rows, n, k, dw, db));
        CK(guard(dx));
        return linear_bwd(x, w, dy, rows, n, k, dx, nullptr, nullptr, m.gws, m.gws_bytes, sv());
    }
    // MLP fc2 backward: dH = (dY W) * GELU'(pre) on the main stream (the activation's VJP in the
    // GEMM epilogue), dW / db on the side stream
    int bwd_xw_gelu(const bf16* x, const bf16* w, const bf16* dy, int64_t rows, int64_t n, int64_t k, const bf16* pre,
                    bf16* dh, float* dw, float* db) const {
        if (!overlap) {
            CK(linear_bwd(x, w, dy, rows, n, k, nullptr, dw, db, m.gws, m.gws_bytes, sv()));
        } else {
            CK(side_dw(x, w, dy, rows, n, k, dw, db));
            CK(guard(dh));
        }
        return linear_dx_gelu(dy, w, pre, rows, n, k, dh, sv());
    }
    // main stream waits for every side-stream weight gradient
    int join() const {
        if (!overlap) return AFFMAE_OK;
        cudaEvent_t e = event();
        if (!e) return fail(AFFMAE_ECUDA, "model: event pool exhausted");
        if (cudaEventRecord(e, m.side) != cudaSuccess || cudaStreamWaitEvent(st, e, 0) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model side join");
        pending.clear();
        return AFFMAE_OK;
    }
    // y = x W^T (+ b); W [n, k] (arena layout of a transposed parameter)
    int fwd(const bf16* x, int64_t rows, int64_t k, const bf16* w, int64_t n, const float* b, bf16* y) const {
        return linear_fwd(x, w, b ? b : m.zero_bias, rows, n, k, 0, y, m.gws, m.gws_bytes, sv());
    }
    // y = GELU(x W^T + b) with the pre-activation kept for the backward: both written by the
    // GEMM's epilogue (gemm_tc.cu kGeluAux)
    int fwd_gelu(const bf16* x, int64_t rows, int64_t k, const bf16* w, int64_t n, const float* b, bf16* y,
                 bf16* pre) const {
        return linear_fwd_gelu_aux(x, w, b, rows, n, k, y, pre, m.gws, m.gws_bytes, sv());
    }
    int fwd_add(const bf16* x, int64_t rows, int64_t k, const bf16* w, int64_t n, const float* b, const bf16* c,
                bf16* y) const {
        return linear_fwd_add(x, w, b, rows, n, k, c, y, m.gws, m.gws_bytes, sv());
    }
    // dW (+db) += from x [rows, k], dy [rows, n]
    int bwd_w(const bf16* x, const bf16* w, const bf16* dy, int64_t rows, int64_t n, int64_t k, float* dw,
              float* db) const {
        return linear_bwd(x, w, dy, rows, n, k, nullptr, dw, db, m.gws, m.gws_bytes, sv());
    }
    int bwd_wx(const bf16* x, const bf16* w, const bf16* dy, int64_t rows, int64_t n, int64_t k, bf16* dx, float* dw,
               float* db) const {
        return linear_bwd(x, w, dy, rows, n, k, dx, dw, db, m.gws, m.gws_bytes, sv());
    }
    // dx (fp32) = dy W (+ beta dx)
    int bwd_x(const bf16* dy, const bf16* w, int64_t rows, int64_t n, int64_t k, float* dx, float beta) const {
        return linear_dx_f32(dy, w, rows, n, k, dx, beta, m.gws, m.gws_bytes, sv());
    }
};

std::string blk_name(int s, int b) { return "enc.s" + std::to_string(s) + ".b" + std::to_string(b) + "."; }
std::string dec_name(int s, int r) { return "dec.s" + std::to_string(s) + ".r" + std::to_string(r) + "."; }

affmae_attn_inputs attn_in(Model& m, const std::string& pre, const bf16* q, const bf16* k, const bf16* v,
                           const float* coords) {
    affmae_attn_inputs in;
    in.q = reinterpret_cast<const affmae_bf16*>(q);
    in.k = reinterpret_cast<const affmae_bf16*>(k);
    in.v = reinterpret_cast<const affmae_bf16*>(v);
    in.blank_k = reinterpret_cast<const affmae_bf16*>(PBF(m, pre + "blank_k"));
    in.blank_v = reinterpret_cast<const affmae_bf16*>(PBF(m, pre + "blank_v"));
    in.coords = coords;
    in.w1 = PF(m, pre + "bias.w1");
    in.b1 = PF(m, pre + "bias.b1");
    in.w2 = PF(m, pre + "bias.w2");
    in.b2 = PF(m, pre + "bias.b2");
    in.blank = PF(m, pre + "bias.blank");
    return in;
}
affmae_attn_grads attn_g(Model& m, const std::string& pre, bf16* dq, bf16* dk, bf16* dv) {
    affmae_attn_grads g;
    g.dq = reinterpret_cast<affmae_bf16*>(dq);
    g.dk = reinterpret_cast<affmae_bf16*>(dk);
    g.dv = reinterpret_cast<affmae_bf16*>(dv);
    g.dblank_k = GF(m, pre + "blank_k");
    g.dblank_v = GF(m, pre + "blank_v");
    g.dw1 = GF(m, pre + "bias.w1");
    g.db1 = GF(m, pre + "bias.b1");
    g.dw2 = GF(m, pre + "bias.w2");
    g.db2 = GF(m, pre + "bias.b2");
    g.dblank = GF(m, pre + "bias.blank");
    return g;
}

// ------------------------------------------------------------------ forward
int block_fwd(const Ctx& x, int s, int b) {
    Model& m = x.m;
    Stage& S = m.st[size_t(s)];
    Blk& k = S.blk[size_t(b)];
    const std::string pre = blk_name(s, b);
    const int64_t M = S.M, D = S.D;
    // Q, K, V in one GEMM: [wq; wk; wv] are adjacent [D, D] blocks of the shadow arena
    CK(x.fwd(k.h1, M, D, PBF(m, pre + "wq"), 3 * D, nullptr, k.qkv));
    affmae_attn_inputs in = attn_in(m, pre, k.qkv, k.qkv + D, k.qkv + 2 * D, S.coords);
    CK(attn_fwd_planned(&S.geom, &S.desc, &in, &S.plan, reinterpret_cast<affmae_bf16*>(k.a), k.lse, m.ws, m.ws_bytes,
                        x.sv(), 3 * D));
    CK(x.fwd(k.a, M, D, PBF(m, pre + "wo"), D, nullptr, m.T1));
    CK(mk::ln_fwd(S.f[size_t(b)], m.T1, k.fmid, nullptr, PF(m, pre + "ln2.g"), PF(m, pre + "ln2.b"), M, D, k.h2, k.st2,
                  x.st));
    CK(x.fwd_gelu(k.h2, M, D, PBF(m, pre + "mlp.w1"), 4 * D, PF(m, pre + "mlp.b1"), k.m, k.pre));
    CK(x.fwd(k.m, M, 4 * D, PBF(m, pre + "mlp.w2"), D, PF(m, pre + "mlp.b2"), m.T1));
    if (b + 1 < int(S.blk.size())) {
        const std::string nx = blk_name(s, b + 1);
        Blk& n = S.blk[size_t(b + 1)];
        return mk::ln_fwd(k.fmid, m.T1, S.f[size_t(b + 1)], nullptr, PF(m, nx + "ln1.g"), PF(m, nx + "ln1.b"), M, D,
                          n.h1, n.st1, x.st);
    }
    return mk::ln_fwd(k.fmid, m.T1, S.f[size_t(b + 1)], S.fout_bf, nullptr, nullptr, M, D, nullptr, nullptr, x.st);
}

int merge_fwd(const Ctx& x, int s) {
    Model& m = x.m;
    const affmae_model_cfg& c = m.cfg;
    Stage& S = m.st[size_t(s)];
    Stage& Sn = m.st[size_t(s + 1)];
    const std::string pre = "merge.s" + std::to_string(s) + ".";
    const int64_t M = S.M, D = S.D, R = S.R, Dn = Sn.D, Mn = m.B * R;
    CK(x.fwd_gelu(S.fout_bf, M, D, PBF(m, pre + "scorer.w1"), 16, PF(m, pre + "scorer.b1"), S.shid, S.spre));
    CK(mk::scorer_out_fwd(S.shid, M, PF(m, pre + "scorer.w2"), PF(m, pre + "scorer.b2"), S.scores, x.st));
    if (S.forced) {
        if (cudaMemcpyAsync(S.ret, S.forced_ret, size_t(m.B * R) * 4, cudaMemcpyDeviceToDevice, x.st) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model forced retained");
    } else {
        CK(select_retained(S.scores, m.B, S.N, c.stages[s].d_s, S.ret, m.ws, m.ws_bytes, x.sv()));
    }
    CK(merge_plan_build(S.coords, S.ret, m.B, S.N, R, c.merge_k, &S.mplan, m.ws, m.ws_bytes, x.sv()));
    CK(merge_pool_fwd(reinterpret_cast<const affmae_bf16*>(S.fout_bf), S.scores, PF(m, pre + "p"), S.ret, &S.mplan,
                      m.B, S.N, R, D, c.merge_k, reinterpret_cast<affmae_bf16*>(S.pooled), x.sv()));
    CK(x.fwd(S.pooled, Mn, 2 * D, PBF(m, pre + "proj"), Dn, nullptr, S.ymerge));
    CK(mk::ln_fwd_bf(S.ymerge, nullptr, PF(m, pre + "ln.g"), PF(m, pre + "ln.b"), Mn, Dn, S.ylnm, S.stm, x.st));
    CK(mk::gather_coords(S.coords, S.ret, m.B, S.N, R, Sn.coords, x.st));
    const std::string nx = blk_name(s + 1, 0);
    return mk::ln_fwd_bf(S.ylnm, Sn.f[0], PF(m, nx + "ln1.g"), PF(m, nx + "ln1.b"), Mn, Dn, Sn.blk[0].h1,
                         Sn.blk[0].st1, x.st);
}

int round_fwd(const Ctx& x, int si, int r, bool last) {
    Model& m = x.m;
    const affmae_model_cfg& c = m.cfg;
    Stage& S = m.st[size_t(si)];
    DecStage& d = m.dec[size_t(si)];
    DecRound& R = d.rounds[size_t(r)];
    const std::string pre = dec_name(si, r);
    const int64_t Mq = m.Mq, dd = m.dd, B = m.B, Q = m.Q;
    affmae_attn_desc desc{c.dec_heads, int(dd / c.dec_heads), c.bias_hidden, double(c.patch)};
    CK(mk::offset_fwd(R.fq_in, Mq, dd, PF(m, pre + "off.w"), PF(m, pre + "off.b"), 2.0 * double(c.patch), m.refs,
                      R.offpre, R.qpos, x.st));
    CK(knn(R.qpos, S.coords, B, Q, S.N, c.gather_k, R.gidx, R.gval, x.sv()));
    CK(interp_fwd(R.qpos, S.coords, d.z, R.gidx, R.gval, B, Q, S.N, dd, c.gather_k, PF(m, pre + "p"), kInterpEps,
                  R.virt, x.sv()));
    CK(mk::ln_fwd(R.fq_in, nullptr, nullptr, nullptr, PF(m, pre + "ln1.g"), PF(m, pre + "ln1.b"), Mq, dd, R.h1, R.st1,
                  x.st));
    CK(x.fwd(R.h1, Mq, dd, PBF(m, pre + "x.wq"), dd, nullptr, R.q1));
    // wk | wv are adjacent in the arena (create checks): one [2dd, dd] projection
    CK(x.fwd(R.virt, Mq, dd, PBF(m, pre + "x.wk"), 2 * dd, nullptr, R.kv1));
    affmae_attn_inputs in1 = attn_in(m, pre + "x.", R.q1, R.kv1, R.kv1 + dd, m.refs);
    CK(gattn_fwd(&desc, &in1, m.one_idx, m.one_val, B, Q, 1, R.a1, R.lse1, x.sv(), dd, 2 * dd));
    CK(x.fwd(R.a1, Mq, dd, PBF(m, pre + "x.wo"), dd, nullptr, m.T1));
    CK(mk::ln_fwd(R.fq_in, m.T1, R.fq_x, nullptr, PF(m, pre + "ln2.g"), PF(m, pre + "ln2.b"), Mq, dd, R.h2, R.st2,
                  x.st));
    CK(x.fwd(R.h2, Mq, dd, PBF(m, pre + "s.wq"), 3 * dd, nullptr, R.qkv2));  // wq | wk | wv
    affmae_attn_inputs in2 = attn_in(m, pre + "s.", R.qkv2, R.qkv2 + dd, R.qkv2 + 2 * dd, m.refs);
    CK(gattn_fwd(&desc, &in2, m.self_idx, m.self_val, B, Q, c.self_k, R.a2, R.lse2, x.sv(), 3 * dd, 3 * dd));
    CK(x.fwd(R.a2, Mq, dd, PBF(m, pre + "s.wo"), dd, nullptr, m.T1));
    CK(mk::ln_fwd(R.fq_x, m.T1, R.fq_s, nullptr, PF(m, pre + "ln3.g"), PF(m, pre + "ln3.b"), Mq, dd, R.h3, R.st3,
                  x.st));
    CK(x.fwd_gelu(R.h3, Mq, dd, PBF(m, pre + "mlp.w1"), 2 * dd, PF(m, pre + "mlp.b1"), R.m, R.pre));
    CK(x.fwd(R.m, Mq, 2 * dd, PBF(m, pre + "mlp.w2"), dd, PF(m, pre + "mlp.b2"), m.T1));
    if (last)
        return mk::ln_fwd(R.fq_s, m.T1, R.fq_out, nullptr, PF(m, "dec.head.ln.g"), PF(m, "dec.head.ln.b"), Mq, dd,
                          m.hh, m.sth, x.st);
    return mk::add_f32_bf16(R.fq_s, 0, m.T1, Mq, dd, R.fq_out, nullptr, x.st);
}

int forward(const Ctx& x) {
    Model& m = x.m;
    const affmae_model_cfg& c = m.cfg;
    const int64_t B = m.B, p2 = m.p2;
    const float inv_image = float(1.0 / double(c.image));
    const bool aux_on = c.lambda_aux > 0.0;
    // Work that depends only on coordinates -- the decoder's self knn over the masked cells and
    // the deep-supervision knn of every stage -- and the deep-supervision heads themselves
    // (interpolation + head GEMM, which read a finished encoder stage) run on the side stream
    // beside the encoder / decoder: forked by events after their inputs are produced, joined
    // before their first main-stream reader (the decoder's self attention, the loss).
    cudaStream_t ss = m.side ? m.side : x.st;
    auto fork = [&]() -> int {
        if (!m.side) return AFFMAE_OK;
        cudaEvent_t e = x.event();
        if (!e) return fail(AFFMAE_ECUDA, "model: event pool exhausted");
        if (cudaEventRecord(e, x.st) != cudaSuccess || cudaStreamWaitEvent(ss, e, 0) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model forward fork");
        return AFFMAE_OK;
    };
    auto join = [&]() -> int {
        if (!m.side) return AFFMAE_OK;
        cudaEvent_t e = x.event();
        if (!e) return fail(AFFMAE_ECUDA, "model: event pool exhausted");
        if (cudaEventRecord(e, ss) != cudaSuccess || cudaStreamWaitEvent(x.st, e, 0) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model forward join");
        return AFFMAE_OK;
    };
    auto aux_knn = [&](int s) -> int {
        Stage& S = m.st[size_t(s)];
        return knn(m.refs, S.coords, B, m.Q, S.N, c.stages[s].interp_k, S.aidx, S.aval, reinterpret_cast<void*>(ss));
    };
    auto aux_head = [&](int s) -> int {
        Stage& S = m.st[size_t(s)];
        const std::string pre = "aux.s" + std::to_string(s) + ".";
        const int k = c.stages[s].interp_k;
        CK(interp_fwd(m.refs, S.coords, S.fout_bf, S.aidx, S.aval, B, m.Q, S.N, S.D, k, PF(m, pre + "p"), kInterpEps,
                      S.avirt, reinterpret_cast<void*>(ss)));
        return linear_fwd(S.avirt, PBF(m, pre + "w"), PF(m, pre + "b"), m.Mq, p2, S.D, 0, S.aout, m.gws,
                          m.gws_bytes, reinterpret_cast<void*>(ss));
    };
    // inputs: patches, visible / masked cells (pipeline.cpp:402-427, 477-492)
    CK(patchify(m.images, B, m.S, m.S, c.patch, m.patches, x.sv()));
    Stage& S0 = m.st[0];
    CK(mk::cell_rows(m.masked, B, m.g, m.g, 0, m.N[0], double(c.patch), m.vis_rows, S0.coords, x.st));
    CK(mk::cell_rows(m.masked, B, m.g, m.g, 1, m.Q, double(c.patch), m.msk_rows, m.refs, x.st));
    CK(fork());
    CK(knn(m.refs, m.refs, B, m.Q, m.Q, c.self_k, m.self_idx, m.self_val, reinterpret_cast<void*>(ss)));
    if (aux_on && m.ns > 1) CK(aux_knn(0));
    CK(mk::gather_rows_bf16(m.patches, m.vis_rows, S0.M, p2, m.vec, x.st));
    // embed + pos_encode (pipeline.cpp:429-433)
    CK(mk::pos_hidden_fwd(S0.coords, S0.M, inv_image, PF(m, "pos0.w1"), PF(m, "pos0.b1"), m.h0, x.st));
    CK(x.fwd(m.h0, S0.M, kPosHidden, PBF(m, "pos0.w2"), S0.D, PF(m, "pos0.b2"), m.ypos0));
    CK(x.fwd_add(m.vec, S0.M, p2, PBF(m, "embed.w"), S0.D, PF(m, "embed.b"), m.ypos0, m.emb));
    CK(mk::ln_fwd_bf(m.emb, S0.f[0], PF(m, blk_name(0, 0) + "ln1.g"), PF(m, blk_name(0, 0) + "ln1.b"), S0.M, S0.D,
                     S0.blk[0].h1, S0.blk[0].st1, x.st));
    // stages (pipeline.cpp:436-469)
    for (int s = 0; s < m.ns; ++s) {
        Stage& S = m.st[size_t(s)];
        CK(cluster_index_build(&S.geom, S.coords, &S.idx, m.ws, m.ws_bytes, x.sv()));
        CK(attn_plan_build(&S.geom, &S.desc, S.coords, &S.idx, 1, &S.plan, x.sv()));
        for (int b = 0; b < int(S.blk.size()); ++b) CK(block_fwd(x, s, b));
        if (aux_on && s + 1 < m.ns) {
            CK(fork());  // the stage output is final: its deep-supervision head runs beside the rest
            CK(aux_head(s));
        }
        if (s + 1 < m.ns) {
            CK(merge_fwd(x, s));
            if (aux_on && s + 2 < m.ns) {
                CK(fork());  // the next stage's coordinates are known
                CK(aux_knn(s + 1));
            }
        }
    }
    // decoder (pipeline.cpp:473-547)
    const int64_t Mq = m.Mq, dd = m.dd;
    CK(mk::pos_hidden_fwd(m.refs, Mq, inv_image, PF(m, "dec.pos.w1"), PF(m, "dec.pos.b1"), m.hq, x.st));
    CK(x.fwd(m.hq, Mq, kPosHidden, PBF(m, "dec.pos.w2"), dd, PF(m, "dec.pos.b2"), m.yposq));
    CK(mk::add_f32_bf16(PF(m, "dec.mask_token"), 1, m.yposq, Mq, dd, m.fq0, nullptr, x.st));
    CK(join());  // self knn (and everything the side stream has so far) before the decoder
    for (int si = m.ns - 1; si >= 0; --si) {
        Stage& S = m.st[size_t(si)];
        DecStage& d = m.dec[size_t(si)];
        const std::string sp = "dec.s" + std::to_string(si) + ".";
        CK(mk::pos_hidden_fwd(S.coords, S.M, inv_image, PF(m, "dec.pos.w1"), PF(m, "dec.pos.b1"), d.hz, x.st));
        CK(x.fwd(d.hz, S.M, kPosHidden, PBF(m, "dec.pos.w2"), dd, PF(m, "dec.pos.b2"), d.zpos));
        CK(x.fwd_add(S.fout_bf, S.M, S.D, PBF(m, sp + "in.w"), dd, PF(m, sp + "in.b"), d.zpos, d.z));
        for (int r = 0; r < c.dec_depth; ++r) CK(round_fwd(x, si, r, si == 0 && r + 1 == c.dec_depth));
    }
    CK(x.fwd(m.hh, Mq, dd, PBF(m, "dec.head.w"), p2, PF(m, "dec.head.b"), m.recon));
    // deep supervision (pipeline.cpp:549-579): the heads ran on the side stream (above)
    const int n_aux = aux_on ? m.ns - 1 : 0;
    CK(join());
    // loss_parts (pipeline.cpp:581-610): the mse gradients are written here too
    // gradient seed 1/world: after the sum over ranks the gradient is that of the GLOBAL batch mean
    const double seed = 1.0 / double(m.world);
    CK(masked_mse(m.recon, m.patches, m.msk_rows, Mq, p2, m.loss + 1, m.drecon, float(seed), m.ws, m.ws_bytes,
                  x.sv()));
    for (int s = 0; s < n_aux; ++s) {
        Stage& S = m.st[size_t(s)];
        CK(masked_mse(S.aout, m.patches, m.msk_rows, Mq, p2, m.loss + 3 + s, S.daux,
                      float(seed * c.lambda_aux / double(n_aux)), m.ws, m.ws_bytes, x.sv()));
    }
    loss_combine_kernel<<<1, 1, 0, x.st>>>(m.loss, n_aux, float(c.lambda_aux));
    AFFMAE_LAUNCH_CHECK("loss_combine_kernel");
    return AFFMAE_OK;
}

// ----------------------------------------------------------------- backward
// df / dfbf hold the gradient of the block's output on entry, of its input on exit.
int block_bwd(const Ctx& x, int s, int b) {
    Model& m = x.m;
    Stage& S = m.st[size_t(s)];
    Blk& k = S.blk[size_t(b)];
    const std::string pre = blk_name(s, b);
    const int64_t M = S.M, D = S.D;
    // MLP branch: out = fmid + GELU(h2 W1 + b1) W2 + b2
    // (weight gradients fork to the side stream; dy buffers alternate dfbf -> dfbf2 -> dfbf and
    // dm (B4) / dqkv (B4b) so the next writer rarely waits for them)
    CK(x.bwd_xw_gelu(k.m, PBF(m, pre + "mlp.w2"), m.dfbf, M, D, 4 * D, k.pre, m.B4, GF(m, pre + "mlp.w2"),
                     GF(m, pre + "mlp.b2")));
    CK(x.side_dw(k.h2, PBF(m, pre + "mlp.w1"), m.B4, M, 4 * D, D, GF(m, pre + "mlp.w1"), GF(m, pre + "mlp.b1")));
    CK(x.bwd_x(m.B4, PBF(m, pre + "mlp.w1"), M, 4 * D, D, m.F1, 0.f));
    CK(x.guard(m.dfbf2));
    CK(mk::ln_bwd(m.F1, k.fmid, k.st2, PF(m, pre + "ln2.g"), M, D, S.df, S.df, m.dfbf2, GF(m, pre + "ln2.g"),
                  GF(m, pre + "ln2.b"), m.part, x.st));
    // attention branch: fmid = f + attn(h1 Wq, h1 Wk, h1 Wv) Wo
    CK(x.bwd_xw(k.a, PBF(m, pre + "wo"), m.dfbf2, M, D, D, m.B1, GF(m, pre + "wo"), nullptr));
    affmae_attn_inputs in = attn_in(m, pre, k.qkv, k.qkv + D, k.qkv + 2 * D, S.coords);
    // dQ | dK | dV interleaved in one [M, 3D] buffer: one dX GEMM (K = 3D), one dW GEMM (N = 3D)
    CK(x.guard(m.B4b));
    affmae_attn_grads g = attn_g(m, pre, m.B4b, m.B4b + D, m.B4b + 2 * D);
    CK(attn_bwd_planned(&S.geom, &S.desc, &in, &S.plan, reinterpret_cast<const affmae_bf16*>(k.a), k.lse,
                        reinterpret_cast<const affmae_bf16*>(m.B1), &g, m.ws, m.ws_bytes, x.sv(), 3 * D));
    CK(x.side_dw(k.h1, PBF(m, pre + "wq"), m.B4b, M, 3 * D, D, GF(m, pre + "wq"), nullptr));
    CK(x.bwd_x(m.B4b, PBF(m, pre + "wq"), M, 3 * D, D, m.F1, 0.f));
    CK(x.guard(m.dfbf));
    return mk::ln_bwd(m.F1, S.f[size_t(b)], k.st1, PF(m, pre + "ln1.g"), M, D, S.df, S.df, m.dfbf,
                      GF(m, pre + "ln1.g"), GF(m, pre + "ln1.b"), m.part, x.st);
}

// stage s+1's input gradient (st[s+1].df) -> merge s -> += st[s].df
int merge_bwd(const Ctx& x, int s) {
    Model& m = x.m;
    const affmae_model_cfg& c = m.cfg;
    Stage& S = m.st[size_t(s)];
    Stage& Sn = m.st[size_t(s + 1)];
    const std::string pre = "merge.s" + std::to_string(s) + ".";
    const int64_t M = S.M, D = S.D, R = S.R, Dn = Sn.D, Mn = m.B * R;
    // f_next = LN(pooled Wproj): dy of the projection (bf16)
    CK(x.guard(m.B4));
    CK(x.guard(m.B2));
    CK(mk::ln_bwd_bf(Sn.df, S.ymerge, S.stm, PF(m, pre + "ln.g"), Mn, Dn, nullptr, nullptr, m.B1, GF(m, pre + "ln.g"),
                     GF(m, pre + "ln.b"), m.part, x.st));
    CK(x.bwd_wx(S.pooled, PBF(m, pre + "proj"), m.B1, Mn, Dn, 2 * D, m.B4, GF(m, pre + "proj"), nullptr));
    CK(merge_pool_bwd(reinterpret_cast<const affmae_bf16*>(S.fout_bf), S.scores, PF(m, pre + "p"), S.ret, &S.mplan,
                      m.B, S.N, R, D, c.merge_k, reinterpret_cast<const affmae_bf16*>(m.B4),
                      reinterpret_cast<affmae_bf16*>(m.B1), m.dscores, GF(m, pre + "p"), m.ws, m.ws_bytes, x.sv()));
    CK(mk::add_f32_bf16(S.df, 0, m.B1, M, D, S.df, nullptr, x.st));
    // scorer: scores = sigmoid(GELU(f W1 + b1) w2 + b2)
    CK(mk::scorer_out_bwd(S.shid, S.scores, m.dscores, M, PF(m, pre + "scorer.w2"), m.B2, GF(m, pre + "scorer.w2"),
                          GF(m, pre + "scorer.b2"), m.part, x.st));
    CK(gelu_bwd(S.spre, m.B2, M * 16, m.B2, x.sv()));
    CK(x.bwd_x(m.B2, PBF(m, pre + "scorer.w1"), M, 16, D, S.df, 1.f));
    return x.bwd_w(S.fout_bf, PBF(m, pre + "scorer.w1"), m.B2, M, 16, D, GF(m, pre + "scorer.w1"),
                   GF(m, pre + "scorer.b1"));
}

int round_bwd(const Ctx& x, int si, int r) {
    Model& m = x.m;
    const affmae_model_cfg& c = m.cfg;
    Stage& S = m.st[size_t(si)];
    DecStage& d = m.dec[size_t(si)];
    DecRound& R = d.rounds[size_t(r)];
    const std::string pre = dec_name(si, r);
    const int64_t Mq = m.Mq, dd = m.dd, B = m.B, Q = m.Q;
    affmae_attn_desc desc{c.dec_heads, int(dd / c.dec_heads), c.bias_hidden, double(c.patch)};
    // MLP
    // (weight gradients on the side stream; dfq's bf16 copy goes dfq_bf -> dfq_bf2 -> dfq_bf,
    // the cross attention's dq / dk | dv use their own B2x / dkv)
    CK(x.bwd_xw_gelu(R.m, PBF(m, pre + "mlp.w2"), m.dfq_bf, Mq, dd, 2 * dd, R.pre, m.B4, GF(m, pre + "mlp.w2"),
                     GF(m, pre + "mlp.b2")));
    CK(x.side_dw(R.h3, PBF(m, pre + "mlp.w1"), m.B4, Mq, 2 * dd, dd, GF(m, pre + "mlp.w1"), GF(m, pre + "mlp.b1")));
    CK(x.bwd_x(m.B4, PBF(m, pre + "mlp.w1"), Mq, 2 * dd, dd, m.F1, 0.f));
    CK(x.guard(m.dfq_bf2));
    CK(mk::ln_bwd(m.F1, R.fq_s, R.st3, PF(m, pre + "ln3.g"), Mq, dd, m.dfq, m.dfq, m.dfq_bf2, GF(m, pre + "ln3.g"),
                  GF(m, pre + "ln3.b"), m.part, x.st));
    // self attention over the knn rows
    CK(x.bwd_xw(R.a2, PBF(m, pre + "s.wo"), m.dfq_bf2, Mq, dd, dd, m.B1, GF(m, pre + "s.wo"), nullptr));
    CK(cudaMemsetAsync(m.F2, 0, size_t(Mq * dd) * 4, x.st) == cudaSuccess ? 0 : AFFMAE_ECUDA);
    CK(cudaMemsetAsync(m.F3, 0, size_t(Mq * dd) * 4, x.st) == cudaSuccess ? 0 : AFFMAE_ECUDA);
    {
        affmae_attn_inputs in2 = attn_in(m, pre + "s.", R.qkv2, R.qkv2 + dd, R.qkv2 + 2 * dd, m.refs);
        const std::string p = pre + "s.";
        // reverse-CSR gather of dk / dv (no fp32 reductions): 1.85 -> 1.49 ms at B = 16; dq goes
        // straight into the dq | dk | dv buffer of the fused projection's backward
        CK(x.guard(m.dqkv));
        CK(gattn_bwd(&desc, &in2, m.self_idx, m.self_val, B, Q, c.self_k, m.B1, m.dqkv, m.F2, m.F3,
                     GF(m, p + "blank_k"), GF(m, p + "blank_v"), GF(m, p + "bias.w1"), GF(m, p + "bias.b1"),
                     GF(m, p + "bias.w2"), GF(m, p + "bias.b2"), GF(m, p + "bias.blank"), m.ws, m.ws_bytes,
                     x.sv(), 3 * dd, 3 * dd, 3 * dd));
    }
    CK(mk::cast_bf16_2d(m.F2, Mq, dd, m.dqkv + dd, 3 * dd, x.st));
    CK(mk::cast_bf16_2d(m.F3, Mq, dd, m.dqkv + 2 * dd, 3 * dd, x.st));
    // one dW GEMM (N = 3dd) and one dX GEMM (K = 3dd) for the fused q | k | v projection
    CK(x.side_dw(R.h2, PBF(m, pre + "s.wq"), m.dqkv, Mq, 3 * dd, dd, GF(m, pre + "s.wq"), nullptr));
    CK(x.bwd_x(m.dqkv, PBF(m, pre + "s.wq"), Mq, 3 * dd, dd, m.F1, 0.f));
    CK(x.guard(m.dfq_bf));
    CK(mk::ln_bwd(m.F1, R.fq_x, R.st2, PF(m, pre + "ln2.g"), Mq, dd, m.dfq, m.dfq, m.dfq_bf, GF(m, pre + "ln2.g"),
                  GF(m, pre + "ln2.b"), m.part, x.st));
    // cross attention over (virtual token, blank)
    CK(x.bwd_xw(R.a1, PBF(m, pre + "x.wo"), m.dfq_bf, Mq, dd, dd, m.B1, GF(m, pre + "x.wo"), nullptr));
    {   // one-to-one rows: dq, dk, dv straight to bf16 (every key row has exactly one query);
        // dk | dv land in one [Mq, 2dd] buffer, the fused k | v projection's dY
        affmae_attn_inputs in1 = attn_in(m, pre + "x.", R.q1, R.kv1, R.kv1 + dd, m.refs);
        const std::string p = pre + "x.";
        CK(x.guard(m.B2x));
        CK(x.guard(m.dkv));
        CK(gattn_bwd_o2o(&desc, &in1, m.one_idx, m.one_val, B, Q, m.B1, m.B2x, m.dkv, m.dkv + dd,
                         GF(m, p + "blank_k"), GF(m, p + "blank_v"), GF(m, p + "bias.w1"), GF(m, p + "bias.b1"),
                         GF(m, p + "bias.w2"), GF(m, p + "bias.b2"), GF(m, p + "bias.blank"), m.ws, m.ws_bytes,
                         x.sv(), dd, 2 * dd, dd, 2 * dd));
    }
    CK(x.side_dw(R.h1, PBF(m, pre + "x.wq"), m.B2x, Mq, dd, dd, GF(m, pre + "x.wq"), nullptr));
    CK(x.side_dw(R.virt, PBF(m, pre + "x.wk"), m.dkv, Mq, 2 * dd, dd, GF(m, pre + "x.wk"), nullptr));
    CK(x.bwd_x(m.B2x, PBF(m, pre + "x.wq"), Mq, dd, dd, m.F1, 0.f));
    CK(x.bwd_x(m.dkv, PBF(m, pre + "x.wk"), Mq, 2 * dd, dd, m.F4, 0.f));
    // virtual tokens: interpolation of z at the deformed points (gradients into z, p, qpos)
    CK(x.guard(m.B6));
    CK(mk::cast_bf16(m.F4, Mq * dd, m.B6, x.st));
    CK(cudaMemsetAsync(m.dqpos, 0, size_t(Mq * 2) * 4, x.st) == cudaSuccess ? 0 : AFFMAE_ECUDA);
    CK(interp_bwd_gather(R.qpos, S.coords, d.z, R.gidx, R.gval, B, Q, S.N, dd, c.gather_k, PF(m, pre + "p"),
                         kInterpEps, m.B6, m.dz, GF(m, pre + "p"), m.dqpos, m.ws, m.ws_bytes, x.sv()));
    // qpos = refs + NormClamp(fq W_off + b_off): += dfq in place
    CK(mk::offset_bwd(R.fq_in, Mq, dd, PF(m, pre + "off.w"), 2.0 * double(c.patch), R.offpre, m.dqpos, m.dfq,
                      GF(m, pre + "off.w"), GF(m, pre + "off.b"), m.part, x.st));
    CK(x.guard(m.dfq_bf));
    return mk::ln_bwd(m.F1, R.fq_in, R.st1, PF(m, pre + "ln1.g"), Mq, dd, m.dfq, m.dfq, m.dfq_bf, GF(m, pre + "ln1.g"),
                      GF(m, pre + "ln1.b"), m.part, x.st);
}

// positional MLP backward given dy (bf16) of its output rows
int pos_bwd(const Ctx& x, const std::string& pre, const bf16* h, const float* coords, int64_t rows, int64_t D,
            const bf16* dy) {
    Model& m = x.m;
    CK(x.bwd_w(h, PBF(m, pre + ".w2"), dy, rows, D, kPosHidden, GF(m, pre + ".w2"), GF(m, pre + ".b2")));
    CK(x.bwd_x(dy, PBF(m, pre + ".w2"), rows, D, kPosHidden, m.F5, 0.f));
    return mk::pos_hidden_bwd(coords, rows, float(1.0 / double(m.cfg.image)), PF(m, pre + ".w1"), PF(m, pre + ".b1"),
                              m.F5, GF(m, pre + ".w1"), GF(m, pre + ".b1"), m.part, x.st);
}

int backward(const Ctx& x) {
    Model& m = x.m;
    const affmae_model_cfg& c = m.cfg;
    const int64_t Mq = m.Mq, dd = m.dd, p2 = m.p2, B = m.B;
    for (Stage& S : m.st)
        if (cudaMemsetAsync(S.df, 0, size_t(S.M * S.D) * 4, x.st) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model backward memset");
    // decoder head: recon = LN(fq) W + b
    CK(x.side_dw(m.hh, PBF(m, "dec.head.w"), m.drecon, Mq, p2, dd, GF(m, "dec.head.w"), GF(m, "dec.head.b")));
    CK(x.bwd_x(m.drecon, PBF(m, "dec.head.w"), Mq, p2, dd, m.F1, 0.f));
    CK(mk::ln_bwd(m.F1, m.fq_final, m.sth, PF(m, "dec.head.ln.g"), Mq, dd, nullptr, m.dfq, m.dfq_bf,
                  GF(m, "dec.head.ln.g"), GF(m, "dec.head.ln.b"), m.part, x.st));
    // deep-supervision heads -> stage features
    if (c.lambda_aux > 0.0) {
        for (int s = 0; s + 1 < m.ns; ++s) {
            Stage& S = m.st[size_t(s)];
            const std::string pre = "aux.s" + std::to_string(s) + ".";
            const int k = c.stages[s].interp_k;
            CK(x.bwd_xw(S.avirt, PBF(m, pre + "w"), S.daux, Mq, p2, S.D, m.B1, GF(m, pre + "w"), GF(m, pre + "b")));
            CK(interp_bwd_gather(m.refs, S.coords, S.fout_bf, S.aidx, S.aval, B, m.Q, S.N, S.D, k,
                                 PF(m, pre + "p"), kInterpEps, m.B1, S.df, GF(m, pre + "p"), m.dqjunk, m.ws,
                                 m.ws_bytes, x.sv()));
        }
    }
    // decoder stages, reverse of the forward order (shallowest first)
    for (int si = 0; si < m.ns; ++si) {
        Stage& S = m.st[size_t(si)];
        DecStage& d = m.dec[size_t(si)];
        const std::string sp = "dec.s" + std::to_string(si) + ".";
        if (cudaMemsetAsync(m.dz, 0, size_t(S.M * dd) * 4, x.st) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model backward memset");
        for (int r = c.dec_depth - 1; r >= 0; --r) CK(round_bwd(x, si, r));
        // z = f W_in + b_in + pos(coords)
        CK(x.guard(m.B6));
        CK(mk::cast_bf16(m.dz, S.M * dd, m.B6, x.st));
        CK(x.side_dw(S.fout_bf, PBF(m, sp + "in.w"), m.B6, S.M, dd, S.D, GF(m, sp + "in.w"), GF(m, sp + "in.b")));
        CK(x.bwd_x(m.B6, PBF(m, sp + "in.w"), S.M, dd, S.D, S.df, 1.f));
        CK(pos_bwd(x, "dec.pos", d.hz, S.coords, S.M, dd, m.B6));
    }
    // fq0 = mask_token (repeated) + pos(refs)
    CK(mk::colsum_f32(m.dfq, Mq, dd, GF(m, "dec.mask_token"), m.part, x.st));
    CK(pos_bwd(x, "dec.pos", m.hq, m.refs, Mq, dd, m.dfq_bf));
    // encoder stages in reverse
    for (int s = m.ns - 1; s >= 0; --s) {
        Stage& S = m.st[size_t(s)];
        if (s + 1 < m.ns) CK(merge_bwd(x, s));
        CK(x.guard(m.dfbf));
        CK(mk::cast_bf16(S.df, S.M * S.D, m.dfbf, x.st));
        for (int b = int(S.blk.size()) - 1; b >= 0; --b) CK(block_bwd(x, s, b));
    }
    // stage-0 input: f0 = vec W_e + b_e + pos0(coords)
    Stage& S0 = m.st[0];
    CK(x.side_dw(m.vec, PBF(m, "embed.w"), m.dfbf, S0.M, S0.D, p2, GF(m, "embed.w"), GF(m, "embed.b")));
    return pos_bwd(x, "pos0", m.h0, S0.coords, S0.M, S0.D, m.dfbf);
}

int forward_backward(Model& m, cudaStream_t st) {
    Ctx x{m, st};
    if (cudaMemsetAsync(m.G, 0, size_t(m.nvals) * 4, st) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model zero_grads");
    CK(forward(x));
    x.overlap = m.side != nullptr;
    CK(backward(x));
    CK(x.join());
    // the step's one exchange: sum the gradient arena over the data-parallel ranks
    if (m.comm) return nccl_allreduce_sum_f32(m.comm, m.G, m.nvals, st);
    return AFFMAE_OK;
}

int apply_step(Model& m, cudaStream_t st) {
    return adamw_step_dev(&m.cfg.optim, m.step_dev, m.adam_scalars, int64_t(m.params.size()), m.seg_off, m.seg_decay,
                          m.nvals, m.P, m.G, m.M1, m.V1, m.PB, m.nshadow, st);
}

// ------------------------------------------------------------------ create
int validate(const affmae_model_cfg& c) {
    // PipelineConfig::validate (proj/src/config.cpp:37-66)
    if (c.image < 1 || c.patch < 1 || c.image % c.patch != 0)
        return fail(AFFMAE_ECONFIG, "config: image size must be a positive multiple of patch");
    if (c.n_stages < 1) return fail(AFFMAE_ECONFIG, "config: need at least one stage");
    if (c.n_stages > AFFMAE_MAX_STAGES) return fail(AFFMAE_EUNSUPPORTED, "config: too many stages");
    for (int s = 0; s < c.n_stages; ++s) {
        const affmae_stage_cfg& st = c.stages[s];
        const std::string tag = "config: stage " + std::to_string(s);
        if (st.dim < 1 || st.heads < 1 || st.dim % st.heads != 0)
            return fail(AFFMAE_ECONFIG, tag + ": dim must be a positive multiple of heads");
        if (st.blocks < 1) return fail(AFFMAE_ECONFIG, tag + ": blocks must be >= 1");
        if (st.cluster < 1) return fail(AFFMAE_ECONFIG, tag + ": cluster size must be >= 1");
        if (st.groups < 1) return fail(AFFMAE_ECONFIG, tag + ": groups must be >= 1");
        if (!(st.d_s > 0.0 && st.d_s <= 1.0)) return fail(AFFMAE_ECONFIG, tag + ": d_s must be in (0, 1]");
        if (st.interp_k < 1) return fail(AFFMAE_ECONFIG, tag + ": interp_k must be >= 1");
    }
    if (c.dec_dim < 1 || c.dec_heads < 1 || c.dec_dim % c.dec_heads != 0)
        return fail(AFFMAE_ECONFIG, "config: decoder dim must be a positive multiple of decoder heads");
    if (c.dec_depth < 1 || c.gather_k < 1 || c.self_k < 1)
        return fail(AFFMAE_ECONFIG, "config: decoder depth and fan-ins must be >= 1");
    if (!(c.mask_ratio >= 0.0 && c.mask_ratio < 1.0)) return fail(AFFMAE_ECONFIG, "config: mask ratio must be in [0, 1)");
    if (c.mask_strategy != 0 && c.mask_strategy != 1)
        return fail(AFFMAE_ECONFIG, "config: mask strategy must be perlin or random");
    if (c.lambda_aux < 0.0) return fail(AFFMAE_ECONFIG, "config: lambda must be >= 0");
    if (c.optim.warmup < 1) return fail(AFFMAE_ECONFIG, "config: warmup must be >= 1 step");
    if (!(c.optim.lr >= 0.0)) return fail(AFFMAE_ECONFIG, "config: lr must be >= 0");
    if (c.optim.total_steps < 1) return fail(AFFMAE_ECONFIG, "optimizer needs at least one step");
    if (c.bias_hidden < 1 || c.scorer_hidden < 1 || c.merge_k < 1)
        return fail(AFFMAE_ECONFIG, "config: hidden widths and merge fan-in must be >= 1");
    if (c.batch < 1) return fail(AFFMAE_ECONFIG, "config: batch must be >= 1");
    // compiled kernel variants
    auto dim_ok = [](int64_t d) { return d % 64 == 0 && d <= 1024 && (d / 64 <= 4 || d / 64 == 6 || d / 64 == 8 || d / 64 == 12 || d / 64 == 16); };
    for (int s = 0; s < c.n_stages; ++s) {
        const affmae_stage_cfg& st = c.stages[s];
        const int64_t hd = st.dim / st.heads;
        if (!dim_ok(st.dim) || (hd != 16 && hd != 32 && hd != 64))
            return fail(AFFMAE_EUNSUPPORTED, "model: stage dims must be 64*{1,2,3,4,6,8,12,16} with head_dim 16/32/64");
        if (s + 1 < c.n_stages && st.dim > 512)
            return fail(AFFMAE_EUNSUPPORTED, "model: merged / supervised stages up to dim 512");
    }
    const int64_t dhd = c.dec_dim / c.dec_heads;
    if (c.dec_dim != 64 && c.dec_dim != 128 && c.dec_dim != 256 && c.dec_dim != 512)
        return fail(AFFMAE_EUNSUPPORTED, "model: decoder dim must be 64, 128, 256 or 512");
    if (dhd != 16 && dhd != 32 && dhd != 64) return fail(AFFMAE_EUNSUPPORTED, "model: decoder head_dim 16/32/64");
    if (c.scorer_hidden != 16) return fail(AFFMAE_EUNSUPPORTED, "model: scorer_hidden must be 16");
    if (c.patch * c.patch % 8) return fail(AFFMAE_EUNSUPPORTED, "model: patch^2 must be a multiple of 8");
    if (c.self_k > 31 || c.gather_k > 32) return fail(AFFMAE_EUNSUPPORTED, "model: fan-ins above 31 not compiled");
    return AFFMAE_OK;
}

int create(const affmae_model_cfg* cfg, Model** out) {
    if (!cfg || !out) return fail(AFFMAE_ECONFIG, "model_create: null pointer");
    CK(validate(*cfg));
    Model* mp = new Model();
    Model& m = *mp;
    m.cfg = *cfg;
    const affmae_model_cfg& c = m.cfg;
    m.ns = c.n_stages;
    m.B = c.batch;
    m.S = c.image;
    m.g = c.image / c.patch;
    m.cells = m.g * m.g;
    m.p2 = c.patch * c.patch;
    m.dd = c.dec_dim;
    m.Q = std::llround(c.mask_ratio * double(m.cells));
    m.Mq = m.B * m.Q;
    auto bad = [&](int code, const std::string& msg) {
        delete mp;
        return fail(code, msg);
    };
    if (m.Q < 1) return bad(AFFMAE_EUNSUPPORTED, "model: the mask must hide at least one cell per image");
    m.N.push_back(m.cells - m.Q);
    if (m.N[0] < 1) return bad(AFFMAE_ECONFIG, "encode: mask leaves no visible tokens");
    for (int s = 0; s + 1 < m.ns; ++s) m.N.push_back(retained_count_impl(m.N[size_t(s)], c.stages[s].d_s));
    m.st.resize(size_t(m.ns));
    for (int s = 0; s < m.ns; ++s) {
        Stage& S = m.st[size_t(s)];
        const affmae_stage_cfg& sc = c.stages[s];
        S.N = m.N[size_t(s)];
        S.D = sc.dim;
        S.M = m.B * S.N;
        S.heads = sc.heads;
        S.R = s + 1 < m.ns ? m.N[size_t(s + 1)] : 0;
        S.geom = affmae_cluster_geom{m.B, S.N, sc.cluster, sc.groups, 0, 0, 0, 0};
        if (affmae_cluster_geometry(&S.geom)) return bad(AFFMAE_ECONFIG, affmae_last_error());
        if (S.geom.max_size > 16 || S.geom.width > 64)
            return bad(AFFMAE_EUNSUPPORTED, "model: cluster size <= 16 and neighbourhood width <= 64 compiled");
        S.desc = affmae_attn_desc{sc.heads, int(sc.dim / sc.heads), c.bias_hidden, double(c.patch)};
    }
    build_params(m);
    for (const Param& p : m.params)  // fused QKV GEMMs need [wq; wk; wv] adjacent in the arena
        if (p.name.size() > 2 && p.name.compare(p.name.size() - 2, 2, "wq") == 0) {
            const std::string base = p.name.substr(0, p.name.size() - 2);
            const int64_t dd2 = p.r * p.c;
            if (m.params[size_t(m.pidx.at(base + "wk"))].off != p.off + dd2 ||
                m.params[size_t(m.pidx.at(base + "wv"))].off != p.off + 2 * dd2)
                return bad(AFFMAE_ECONFIG, "model: internal parameter layout (q/k/v not adjacent)");
        }
    Arena a;
    layout(m, a);
    const size_t part_f = part_floats(m);
    m.ws_bytes = misc_ws_bytes(m);
    m.gws_bytes = gemm_ws_bytes(m);
    const size_t main_bytes = a.off;
    m.dbytes = main_bytes + ((part_f * 4 + 255) & ~size_t(255)) + ((m.ws_bytes + 255) & ~size_t(255)) +
               2 * ((m.gws_bytes + 255) & ~size_t(255));
    if (cudaMalloc(&m.dmem, m.dbytes) != cudaSuccess) {
        cudaGetLastError();
        return bad(AFFMAE_ECUDA, "model_create: cudaMalloc of " + std::to_string(m.dbytes >> 20) + " MiB failed");
    }
    a = Arena{m.dmem, 0};
    layout(m, a);
    m.part = reinterpret_cast<float*>(m.dmem + main_bytes);
    m.ws = m.dmem + main_bytes + ((part_f * 4 + 255) & ~size_t(255));
    m.gws = m.ws + ((m.ws_bytes + 255) & ~size_t(255));
    m.gws2 = m.gws + ((m.gws_bytes + 255) & ~size_t(255));
    // the side stream of the backward's weight gradients and its fork / join events (two per
    // weight-gradient GEMM at most, plus the joins)
    if (!std::getenv("AFFMAE_NO_DW_OVERLAP")) {
        if (cudaStreamCreateWithFlags(&m.side, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            m.side = nullptr;
        }
        for (size_t i = 0; m.side && i < 2 * m.params.size() + 8 + 4 * size_t(m.ns) + 8; ++i) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaFree(m.dmem);
                return bad(AFFMAE_ECUDA, "model_create: event creation failed");
            }
            m.events.push_back(e);
        }
    }
    for (Stage& S : m.st) {
        S.plan.batch = S.plan.tokens = S.plan.n_clusters = S.plan.groups_eff = S.plan.width = 0;
        S.plan.has_reverse = 0;
    }
    // zero everything (padding rows of activations stay zero), then upload the init
    if (cudaMemset(m.dmem, 0, m.dbytes) != cudaSuccess) {
        cudaFree(m.dmem);
        return bad(AFFMAE_ECUDA, "model_create: memset failed");
    }
    std::vector<float> host(size_t(m.nvals), 0.f);
    std::vector<int64_t> off;
    std::vector<uint8_t> dec;
    for (const Param& p : m.params) to_arena(p, p.init.data(), host.data());
    std::vector<int> order(m.params.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = int(i);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return m.params[size_t(x)].off < m.params[size_t(y)].off; });
    for (int i : order) {
        off.push_back(m.params[size_t(i)].off);
        dec.push_back(m.params[size_t(i)].decay ? 1 : 0);
    }
    for (Param& p : m.params) std::vector<float>().swap(p.init);
    bool ok = cudaMemcpy(m.P, host.data(), size_t(m.nvals) * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(m.seg_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(m.seg_decay, dec.data(), dec.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) {
        mk::shadow_cast(m.P, m.nshadow, m.PB, nullptr);
        fill_one_to_one_kernel<<<256, 256>>>(m.one_idx, m.one_val, m.B, m.Q);
        ok = cudaDeviceSynchronize() == cudaSuccess;
    }
    if (!ok) {
        cudaFree(m.dmem);
        return bad(AFFMAE_ECUDA, "model_create: upload failed");
    }
    *out = mp;
    return AFFMAE_OK;
}

}  // namespace
}  // namespace affmae_b200

using namespace affmae_b200;

#define AFFMAE_MGUARD(...)                                                         \
    try {                                                                          \
        __VA_ARGS__                                                                \
    } catch (const std::exception& e) {                                            \
        return fail(AFFMAE_ECONFIG, std::string("exception: ") + e.what());       \
    } catch (...) {                                                                \
        return fail(AFFMAE_ECONFIG, "unknown exception");                          \
    }

extern "C" {

int affmae_model_create(const affmae_model_cfg* cfg, affmae_model** out) { AFFMAE_MGUARD(return create(cfg, out);) }

void affmae_model_destroy(affmae_model* m) {
    if (!m) return;
    if (m->gexec) cudaGraphExecDestroy(m->gexec);
    if (m->comm) nccl_comm_destroy(m->comm);
    for (cudaEvent_t e : m->events) cudaEventDestroy(e);
    if (m->side) cudaStreamDestroy(m->side);
    if (m->dmem) cudaFree(m->dmem);
    delete m;
}

int affmae_model_get_info(const affmae_model* m, affmae_model_info* info) {
    if (!m || !info) return fail(AFFMAE_ECONFIG, "model_info: null pointer");
    std::memset(info, 0, sizeof(*info));
    info->n_params = int(m->params.size());
    for (const Param& p : m->params) info->n_values += p.r * p.c;
    for (int s = 0; s < m->ns; ++s) info->tokens[s] = m->N[size_t(s)];
    info->masked = m->Q;
    info->device_bytes = int64_t(m->dbytes);
    info->steps_taken = m->steps;
    return AFFMAE_OK;
}

const char* affmae_model_param_name(const affmae_model* m, int i) {
    if (!m || i < 0 || i >= int(m->params.size())) return nullptr;
    return m->params[size_t(i)].name.c_str();
}

int affmae_model_param_dims(const affmae_model* m, int i, int64_t* rows, int64_t* cols) {
    if (!m || i < 0 || i >= int(m->params.size()) || !rows || !cols) return fail(AFFMAE_ECONFIG, "model_param_dims");
    *rows = m->params[size_t(i)].r;
    *cols = m->params[size_t(i)].c;
    return AFFMAE_OK;
}

static int dev_to_ref(affmae_model* m, const float* dev, std::vector<float>& ref);
static int ref_to_dev(affmae_model* m, const float* ref, float* dev);
static int copy_out(affmae_model* m, const float* dev, float* host) {
    std::vector<float> ref;
    if (int rc = dev_to_ref(m, dev, ref)) return rc;
    std::memcpy(host, ref.data(), ref.size() * 4);
    return AFFMAE_OK;
}

int affmae_model_get_params(affmae_model* m, float* host) {
    if (!m || !host) return fail(AFFMAE_ECONFIG, "model_get_params: null pointer");
    AFFMAE_MGUARD(return copy_out(m, m->P, host);)
}
int affmae_model_get_grads(affmae_model* m, float* host) {
    if (!m || !host) return fail(AFFMAE_ECONFIG, "model_get_grads: null pointer");
    AFFMAE_MGUARD(return copy_out(m, m->G, host);)
}
int affmae_model_set_params(affmae_model* m, const float* host) {
    if (!m || !host) return fail(AFFMAE_ECONFIG, "model_set_params: null pointer");
    AFFMAE_MGUARD(
        if (int rc = ref_to_dev(m, host, m->P)) return rc;
        if (int rc = mk::shadow_cast(m->P, m->nshadow, m->PB, nullptr)) return rc;
        if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status(cudaGetLastError(), "model set params");
        return AFFMAE_OK;)
}

int affmae_model_inputs(affmae_model* m, double** images, uint8_t** masked) {
    if (!m) return fail(AFFMAE_ECONFIG, "model_inputs: null model");
    if (images) *images = m->images;
    if (masked) *masked = m->masked;
    return AFFMAE_OK;
}

int affmae_model_make_masks(affmae_model* m, const uint64_t* seeds_host, void* stream) {
    if (!m || !seeds_host) return fail(AFFMAE_ECONFIG, "model_make_masks: null pointer");
    AFFMAE_MGUARD(
        const affmae_model_cfg& c = m->cfg;
        if (c.mask_strategy == 0)
            return perlin_mask(seeds_host, m->B, m->g, m->g, 2, 4.0, 0.5, c.mask_ratio, m->masked, m->ws, m->ws_bytes,
                               stream);
        // random_mask (proj/src/masking.cpp:94-110)
        std::vector<uint8_t> h(size_t(m->B * m->cells), 0);
        for (int64_t b = 0; b < m->B; ++b) {
            std::vector<int64_t> order(size_t(m->cells));
            for (int64_t i = 0; i < m->cells; ++i) order[size_t(i)] = i;
            Rng rng(mix64(seeds_host[b]) ^ 0x6d61736bull);
            for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[size_t(rng.below(i))]);
            for (int64_t i = 0; i < m->Q; ++i) h[size_t(b * m->cells + order[size_t(i)])] = 1;
        }
        if (cudaMemcpyAsync(m->masked, h.data(), h.size(), cudaMemcpyHostToDevice, as_stream(stream)) != cudaSuccess ||
            cudaStreamSynchronize(as_stream(stream)) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model random masks");
        return AFFMAE_OK;)
}

int affmae_model_forward_backward(affmae_model* m, float* loss3, void* stream) {
    if (!m) return fail(AFFMAE_ECONFIG, "model_forward_backward: null model");
    AFFMAE_MGUARD(
        cudaStream_t st = as_stream(stream);
        if (int rc = forward_backward(*m, st)) return rc;
        if (loss3 && cudaMemcpyAsync(loss3, m->loss, 12, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model loss copy");
        return AFFMAE_OK;)
}

int affmae_model_forward(affmae_model* m, float* loss3, void* stream) {
    if (!m) return fail(AFFMAE_ECONFIG, "model_forward: null model");
    AFFMAE_MGUARD(
        cudaStream_t st = as_stream(stream);
        Ctx x{*m, st};
        if (int rc = forward(x)) return rc;
        if (loss3 && cudaMemcpyAsync(loss3, m->loss, 12, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model loss copy");
        return AFFMAE_OK;)
}

int affmae_model_reset_optimizer(affmae_model* m, int64_t total_steps) {
    if (!m) return fail(AFFMAE_ECONFIG, "model_reset_optimizer: null model");
    if (total_steps < 1) return fail(AFFMAE_ECONFIG, "optimizer needs at least one step");
    m->cfg.optim.total_steps = total_steps;
    const int64_t zero = 0;
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemset(m->M1, 0, size_t(m->nvals) * 4) != cudaSuccess ||
        cudaMemset(m->V1, 0, size_t(m->nvals) * 4) != cudaSuccess ||
        cudaMemcpy(m->step_dev, &zero, 8, cudaMemcpyHostToDevice) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model_reset_optimizer");
    m->steps = 0;
    if (m->gexec) {  // the captured step bakes the schedule's total_steps
        cudaGraphExecDestroy(m->gexec);
        m->gexec = nullptr;
    }
    return AFFMAE_OK;
}

int affmae_model_apply_step(affmae_model* m, void* stream) {
    if (!m) return fail(AFFMAE_ECONFIG, "model_apply_step: null model");
    AFFMAE_MGUARD(
        if (int rc = apply_step(*m, as_stream(stream))) return rc;
        ++m->steps;
        return AFFMAE_OK;)
}

int affmae_model_train_step(affmae_model* m, float* loss3, int use_graph, void* stream) {
    if (!m) return fail(AFFMAE_ECONFIG, "model_train_step: null model");
    AFFMAE_MGUARD(
        cudaStream_t st = as_stream(stream);
        if (!use_graph) {
            if (int rc = forward_backward(*m, st)) return rc;
            if (int rc = apply_step(*m, st)) return rc;
        } else {
            if (m->gexec && m->gstream != st) {
                cudaGraphExecDestroy(m->gexec);
                m->gexec = nullptr;
            }
            if (!m->gexec) {
                if (!st) return fail(AFFMAE_ECONFIG, "model_train_step: graph mode needs a non-default stream");
                cudaGraph_t g = nullptr;
                if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
                    return cuda_status(cudaGetLastError(), "model graph capture");
                int rc = forward_backward(*m, st);
                if (!rc) rc = apply_step(*m, st);
                const cudaError_t e = cudaStreamEndCapture(st, &g);
                if (rc) {
                    if (g) cudaGraphDestroy(g);
                    return rc;
                }
                if (e != cudaSuccess) return cuda_status(e, "model graph capture");
                const cudaError_t ie = cudaGraphInstantiate(&m->gexec, g, 0);
                cudaGraphDestroy(g);
                if (ie != cudaSuccess) return cuda_status(ie, "model graph instantiate");
                m->gstream = st;
            }
            if (cudaGraphLaunch(m->gexec, st) != cudaSuccess) return cuda_status(cudaGetLastError(), "model graph launch");
        }
        ++m->steps;
        if (loss3 && cudaMemcpyAsync(loss3, m->loss, 12, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model loss copy");
        return AFFMAE_OK;)
}

int affmae_model_stage_output(affmae_model* m, int stage, float* coords_host, float* feats_host,
                              float* scores_host) {
    if (!m || stage < 0 || stage >= m->ns) return fail(AFFMAE_ECONFIG, "model_stage_output: bad stage");
    const Stage& S = m->st[size_t(stage)];
    if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status(cudaGetLastError(), "model_stage_output");
    if (coords_host && cudaMemcpy(coords_host, S.coords, size_t(S.M) * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model_stage_output");
    if (feats_host && cudaMemcpy(feats_host, S.f.back(), size_t(S.M * S.D) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model_stage_output");
    if (scores_host && S.scores &&
        cudaMemcpy(scores_host, S.scores, size_t(S.M) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model_stage_output");
    return AFFMAE_OK;
}

int affmae_model_force_retained(affmae_model* m, int stage, const int32_t* retained_host) {
    if (!m || stage < 0 || stage + 1 >= m->ns) return fail(AFFMAE_ECONFIG, "model_force_retained: bad stage");
    Stage& S = m->st[size_t(stage)];
    if (!retained_host) {
        S.forced = false;
        return AFFMAE_OK;
    }
    for (int64_t b = 0; b < m->B; ++b)
        for (int64_t i = 0; i < S.R; ++i) {
            const int32_t v = retained_host[b * S.R + i];
            if (v < 0 || v >= S.N || (i && v <= retained_host[b * S.R + i - 1]))
                return fail(AFFMAE_ECONFIG, "model_force_retained: indices must be ascending and in range");
        }
    if (cudaMemcpy(S.forced_ret, retained_host, size_t(m->B * S.R) * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model_force_retained");
    S.forced = true;
    return AFFMAE_OK;
}

int affmae_nccl_unique_id(uint8_t* out128) { AFFMAE_MGUARD(return nccl_unique_id(out128);) }

int affmae_model_set_world(affmae_model* m, int world, int rank, const uint8_t* nccl_id) {
    if (!m || world < 1 || rank < 0 || rank >= world) return fail(AFFMAE_ECONFIG, "model_set_world: bad arguments");
    AFFMAE_MGUARD(
        if (m->comm) {
            nccl_comm_destroy(m->comm);
            m->comm = nullptr;
        }
        // (a one-rank communicator is allowed: it runs the same captured exchange, a no-op sum)
        if (nccl_id)
            if (int rc = nccl_comm_init(nccl_id, world, rank, &m->comm)) return rc;
        m->world = world;
        if (m->gexec) {  // the captured step bakes the loss seed and the exchange
            cudaGraphExecDestroy(m->gexec);
            m->gexec = nullptr;
        }
        return AFFMAE_OK;)
}

int affmae_model_grad_buffer(affmae_model* m, float** grad, int64_t* n) {
    if (!m || !grad || !n) return fail(AFFMAE_ECONFIG, "model_grad_buffer: null pointer");
    *grad = m->G;
    *n = m->nvals;
    return AFFMAE_OK;
}

// arena (device) <-> concatenated reference-layout host values
static int dev_to_ref(affmae_model* m, const float* dev, std::vector<float>& ref) {
    std::vector<float> host(size_t(m->nvals));
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(host.data(), dev, size_t(m->nvals) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model copy out");
    int64_t total = 0;
    for (const Param& p : m->params) total += p.r * p.c;
    ref.assign(size_t(total), 0.f);
    int64_t o = 0;
    for (const Param& p : m->params) {
        from_arena(p, host.data(), ref.data() + o);
        o += p.r * p.c;
    }
    return AFFMAE_OK;
}
static int ref_to_dev(affmae_model* m, const float* ref, float* dev) {
    std::vector<float> a(size_t(m->nvals), 0.f);
    int64_t o = 0;
    for (const Param& p : m->params) {
        to_arena(p, ref + o, a.data());
        o += p.r * p.c;
    }
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(dev, a.data(), size_t(m->nvals) * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model copy in");
    return AFFMAE_OK;
}

// checkpoint_save / checkpoint_load of `sets` (reference-layout host arrays, one per suffix)
// through a temporary device buffer; optional trailing scalar "step"
struct TmpDev {
    float* p = nullptr;
    ~TmpDev() {
        if (p) cudaFree(p);
    }
};
static int ckpt_io(affmae_model* m, const std::string& dir, std::vector<std::vector<float>*> sets,
                   std::vector<std::string> suffixes, double* step, bool save) {
    int64_t total = 0;
    for (const Param& p : m->params) total += p.r * p.c;
    const size_t n = size_t(total) * sets.size() + 1;
    TmpDev tmp;
    if (cudaMalloc(&tmp.p, n * 4) != cudaSuccess) return cuda_status(cudaGetLastError(), "model checkpoint");
    std::vector<float> flat(n, 0.f);
    if (save) {
        for (size_t k = 0; k < sets.size(); ++k)
            std::memcpy(flat.data() + k * size_t(total), sets[k]->data(), size_t(total) * 4);
        flat[n - 1] = step ? float(*step) : 0.f;
        if (cudaMemcpy(tmp.p, flat.data(), n * 4, cudaMemcpyHostToDevice) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model checkpoint");
    }
    std::vector<std::string> names;
    std::vector<std::vector<int64_t>> dims;
    std::vector<float*> vp;
    std::vector<int64_t> numel;
    for (size_t k = 0; k < sets.size(); ++k) {
        int64_t o = int64_t(k) * total;
        for (const Param& p : m->params) {
            names.push_back(p.name + suffixes[k]);
            dims.push_back({p.r, p.c});
            vp.push_back(tmp.p + o);
            numel.push_back(p.r * p.c);
            o += p.r * p.c;
        }
    }
    if (step) {
        names.push_back("step");
        dims.push_back({1});
        vp.push_back(tmp.p + n - 1);
        numel.push_back(1);
    }
    std::vector<const char*> np;
    std::vector<const int64_t*> dp;
    std::vector<int> nd, pr;
    for (size_t i = 0; i < names.size(); ++i) {
        np.push_back(names[i].c_str());
        dp.push_back(dims[i].data());
        nd.push_back(int(dims[i].size()));
        pr.push_back(0);
    }
    if (save) {
        std::vector<const float*> cvp(vp.begin(), vp.end());
        return checkpoint_save(dir.c_str(), int(names.size()), np.data(), cvp.data(), dp.data(), nd.data(), pr.data(),
                               nullptr);
    }
    if (int rc = checkpoint_load(dir.c_str(), int(names.size()), np.data(), vp.data(), numel.data(), nullptr)) return rc;
    if (cudaMemcpy(flat.data(), tmp.p, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "model checkpoint");
    for (size_t k = 0; k < sets.size(); ++k)
        sets[k]->assign(flat.begin() + int64_t(k) * total, flat.begin() + int64_t(k + 1) * total);
    if (step) *step = double(flat[n - 1]);
    return AFFMAE_OK;
}

int affmae_model_save(affmae_model* m, const char* dir) {
    if (!m || !dir) return fail(AFFMAE_ECONFIG, "model_save: null pointer");
    AFFMAE_MGUARD(
        std::vector<float> p, mo, vo;
        if (int rc = dev_to_ref(m, m->P, p)) return rc;
        if (int rc = ckpt_io(m, dir, {&p}, {""}, nullptr, true)) return rc;
        if (int rc = dev_to_ref(m, m->M1, mo)) return rc;
        if (int rc = dev_to_ref(m, m->V1, vo)) return rc;
        double step = double(m->steps);
        return ckpt_io(m, std::string(dir) + "/optim", {&mo, &vo}, {".m", ".v"}, &step, true);)
}

int affmae_model_load(affmae_model* m, const char* dir) {
    if (!m || !dir) return fail(AFFMAE_ECONFIG, "model_load: null pointer");
    AFFMAE_MGUARD(
        std::vector<float> p, mo, vo;
        if (int rc = ckpt_io(m, dir, {&p}, {""}, nullptr, false)) return rc;
        if (int rc = ref_to_dev(m, p.data(), m->P)) return rc;
        if (int rc = mk::shadow_cast(m->P, m->nshadow, m->PB, nullptr)) return rc;
        const std::string od = std::string(dir) + "/optim";
        FILE* f = std::fopen((od + "/manifest.tsv").c_str(), "rb");
        int64_t steps = 0;
        if (f) {
            std::fclose(f);
            double step = 0;
            if (int rc = ckpt_io(m, od, {&mo, &vo}, {".m", ".v"}, &step, false)) return rc;
            if (int rc = ref_to_dev(m, mo.data(), m->M1)) return rc;
            if (int rc = ref_to_dev(m, vo.data(), m->V1)) return rc;
            steps = int64_t(step);
        } else if (cudaMemset(m->M1, 0, size_t(m->nvals) * 4) != cudaSuccess ||
                   cudaMemset(m->V1, 0, size_t(m->nvals) * 4) != cudaSuccess) {
            return cuda_status(cudaGetLastError(), "model load");
        }
        m->steps = steps;
        if (cudaMemcpy(m->step_dev, &steps, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess)
            return cuda_status(cudaGetLastError(), "model load");
        return AFFMAE_OK;)
}

}  // extern "C"
