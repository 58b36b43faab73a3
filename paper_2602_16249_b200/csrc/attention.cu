// Host side of the cluster attention: validation, workspace layout, BiasNet
// table build, kernel-variant dispatch and the gradient finalisation launches.
// Kernels: attn_kernels.cuh (instantiated per head_dim in attn_inst_d*.cu).
#include <cstdlib>

#include "attn_kernels.cuh"

namespace affmae_b200 {

// ------------------------------------------------------------ bias table
// T[h][(oy+kRg)*kWg + (ox+kRg)] = b2 + sum_u w2 tanh(w1x ox + w1y oy + b1)
// (BiasNet::eval at integer patch offsets, proj/src/attention.cpp:33-42).
__global__ void bias_table_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                  const float* __restrict__ w2, const float* __restrict__ b2,
                                  int heads, int hidden, float* __restrict__ tab) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= heads * kWg2) return;
    int h = i / kWg2, e = i - h * kWg2;
    float ox = float(e % kWg - kRg), oy = float(e / kWg - kRg);
    float acc = b2[h];
    for (int u = 0; u < hidden; ++u) {
        float pre = w1[h * 2 * hidden + u] * ox + w1[h * 2 * hidden + hidden + u] * oy +
                    b1[h * hidden + u];
        acc += w2[h * hidden + u] * tanhf(pre);
    }
    tab[i] = acc;
}

// -------------------------------------------- BiasNet gradient finalize
// dL/dtheta = sum over table entries of dT * dT/dtheta, plus the tier-3
// partials; accumulated (+=) into the caller's gradients.
__global__ void bias_grad_finalize_kernel(const float* __restrict__ dtab, const float* __restrict__ w1,
                                          const float* __restrict__ b1, const float* __restrict__ w2,
                                          int hidden, float* dw1, float* db1, float* dw2, float* db2) {
    const int h = blockIdx.y;
    const float* dt = dtab + size_t(h) * kWg2;
    __shared__ float red[5][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // db2
    {
        float acc = 0.f;
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kWg2; e += gridDim.x * blockDim.x) acc += dt[e];
        acc = warp_sum(acc);
        if (lane == 0) red[0][warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float s = 0.f;
            for (int w = 0; w < nw; ++w) s += red[0][w];
            atomicAdd(db2 + h, s);
        }
        __syncthreads();
    }
    for (int u = 0; u < hidden; ++u) {
        const float wx = w1[h * 2 * hidden + u], wy = w1[h * 2 * hidden + hidden + u];
        const float bb = b1[h * hidden + u], ww = w2[h * hidden + u];
        float gx = 0.f, gy = 0.f, gb = 0.f, gw = 0.f;
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kWg2; e += gridDim.x * blockDim.x) {
            float d = dt[e];
            if (d == 0.f) continue;
            float ox = float(e % kWg - kRg), oy = float(e / kWg - kRg);
            float t = tanhf(wx * ox + wy * oy + bb);
            float dpre = d * ww * (1.f - t * t);
            gx = fmaf(dpre, ox, gx);
            gy = fmaf(dpre, oy, gy);
            gb += dpre;
            gw = fmaf(d, t, gw);
        }
        gx = warp_sum(gx);
        gy = warp_sum(gy);
        gb = warp_sum(gb);
        gw = warp_sum(gw);
        if (lane == 0) {
            red[0][warp] = gx;
            red[1][warp] = gy;
            red[2][warp] = gb;
            red[3][warp] = gw;
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            float s = 0.f;
            for (int w = 0; w < nw; ++w) s += red[threadIdx.x][w];
            float* dst = threadIdx.x == 0 ? dw1 + h * 2 * hidden + u
                       : threadIdx.x == 1 ? dw1 + h * 2 * hidden + hidden + u
                       : threadIdx.x == 2 ? db1 + h * hidden + u
                                          : dw2 + h * hidden + u;
            atomicAdd(dst, s);
        }
        __syncthreads();
    }
}

// tier-3 partials and blank grads -> caller's gradient buffers (+=)
__global__ void attn_grad_epilogue_kernel(const float* __restrict__ mlp_grad,
                                          const float* __restrict__ blank_grad, int heads,
                                          int hidden, int hd, float* dw1, float* db1, float* dw2,
                                          float* db2, float* dbk, float* dbv, float* dblank) {
    const int h = blockIdx.x;
    const float* mg = mlp_grad + h * (4 * hidden + 1);
    const float* bg = blank_grad + h * (2 * hd + 1);
    for (int u = threadIdx.x; u < hidden; u += blockDim.x) {
        dw1[h * 2 * hidden + u] += mg[u];
        dw1[h * 2 * hidden + hidden + u] += mg[hidden + u];
        db1[h * hidden + u] += mg[2 * hidden + u];
        dw2[h * hidden + u] += mg[3 * hidden + u];
    }
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        dbk[h * hd + d] += bg[d];
        dbv[h * hd + d] += bg[hd + d];
    }
    if (threadIdx.x == 0) {
        db2[h] += mg[4 * hidden];
        dblank[h] += bg[2 * hd];
    }
}


template <int HD, int NT, int HPC>
int launch_fwd(const AttnParams& p, cudaStream_t st);
template <int HD, int NT, int HPC>
int launch_bwd(const AttnParams& p, cudaStream_t st);

int pick_nt(int width) {
    int need = (width + 1 + 7) / 8;
    if (need <= 4) return 4;
    if (need <= 7) return 7;
    return -1;
}

static int heads_per_cta(int heads) {
    // AFFMAE_HPC (1, 2 or 4) overrides the head-group width for experiments
    static int force = [] {
        const char* e = getenv("AFFMAE_HPC");
        return e ? atoi(e) : 0;
    }();
    if ((force == 1 || force == 2 || force == 4) && heads % force == 0) return force;
    if (heads % 4 == 0) return 4;
    if (heads % 2 == 0) return 2;
    return 1;
}

static int attn_check(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (!g || !a) return fail(AFFMAE_ECONFIG, "attention: null descriptor");
    if (g->n_clusters <= 0) return fail(AFFMAE_ECONFIG, "attention: geometry not derived (call affmae_cluster_geometry)");
    if (a->heads < 1 || a->head_dim < 1 || a->bias_hidden < 1 || !(a->patch > 0.0))
        return fail(AFFMAE_ECONFIG, "attention: heads, head_dim, bias_hidden, patch must be positive");
    if (a->head_dim != 16 && a->head_dim != 32 && a->head_dim != 64)
        return fail(AFFMAE_EUNSUPPORTED, "attention: head_dim must be 16, 32 or 64");
    if (g->max_size > 16)
        return fail(AFFMAE_EUNSUPPORTED, "attention: clusters larger than 16 tokens not compiled");
    if (pick_nt(int(g->width)) < 0)
        return fail(AFFMAE_EUNSUPPORTED, "attention: neighbourhood width > 55 not compiled");
    if (a->bias_hidden > kMaxHidden) return fail(AFFMAE_EUNSUPPORTED, "attention: bias_hidden > 32");
    return AFFMAE_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct AttnWs {
    float* tab_g;
    int32_t* keylist;
    float* dtab_g;
    float* dsum;
    float* mlp_grad;
    float* blank_grad;
    int32_t* inq;
    size_t bytes;
};

static AttnWs carve_ws(const affmae_cluster_geom* g, const affmae_attn_desc* a, void* base, bool bwd) {
    AttnWs w{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    };
    const size_t items = size_t(g->batch) * g->n_clusters;
    w.tab_g = reinterpret_cast<float*>(take(size_t(a->heads) * kWg2 * 4));
    w.keylist = reinterpret_cast<int32_t*>(take(items * (g->width + 1) * 4));
    if (bwd) {
        w.dtab_g = reinterpret_cast<float*>(take(size_t(a->heads) * kWg2 * 4));
        w.dsum = reinterpret_cast<float*>(take(size_t(g->batch) * g->tokens * a->heads * 4));
        w.mlp_grad = reinterpret_cast<float*>(take(size_t(a->heads) * (4 * a->bias_hidden + 1) * 4));
        w.blank_grad = reinterpret_cast<float*>(take(size_t(a->heads) * (2 * a->head_dim + 1) * 4));
        w.inq = reinterpret_cast<int32_t*>(take(items * g->groups_eff * 16 * 4));
    }
    w.bytes = off;
    return w;
}

// Per cluster: the key token of every neighbourhood slot (reference slot
// order, -1 padding) and, in entry M, the key count nk
// (cluster_neighborhood, proj/src/geometry.cpp:173-183).
__global__ void keylist_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ nbr_cl,
                               ClusterShape cs, int64_t items, int32_t* __restrict__ keylist) {
    const int M = cs.width;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= items * (M + 1)) return;
    int64_t item = i / (M + 1);
    int slot = int(i - item * (M + 1));
    int img = int(item / cs.c);
    const int32_t* nb = nbr_cl + item * cs.g;
    int start = 0, tok = -1;
    for (int g = 0; g < cs.g; ++g) {
        int cl = nb[g], len = cs.len(cl);
        if (slot < M && slot < start + len) {
            tok = perm[int64_t(img) * cs.n + cs.off(cl) + slot - start];
            break;
        }
        start += len;
    }
    keylist[i] = slot == M ? start : tok;
}

// Per reverse pair (CSR order of rev_cl): the query tokens of the pair's query cluster.
__global__ void inq_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ rev_cl,
                           ClusterShape cs, int64_t batch, int32_t* __restrict__ inq) {
    const int64_t pairs = int64_t(cs.c) * cs.g;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= batch * pairs * 16) return;
    int j = int(i & 15);
    int64_t pr = i >> 4;
    int img = int(pr / pairs);
    int c = rev_cl[pr];
    inq[i] = j < cs.len(c) ? perm[int64_t(img) * cs.n + cs.off(c) + j] : -1;
}

static void fill_common(AttnParams& p, const affmae_cluster_geom* g, const affmae_attn_desc* a,
                        const affmae_attn_inputs* in) {
    p = AttnParams{};
    p.q = reinterpret_cast<const __nv_bfloat16*>(in->q);
    p.k = reinterpret_cast<const __nv_bfloat16*>(in->k);
    p.v = reinterpret_cast<const __nv_bfloat16*>(in->v);
    p.bk = reinterpret_cast<const __nv_bfloat16*>(in->blank_k);
    p.bv = reinterpret_cast<const __nv_bfloat16*>(in->blank_v);
    p.coords = in->coords;
    p.w1 = in->w1;
    p.b1 = in->b1;
    p.w2 = in->w2;
    p.b2 = in->b2;
    p.blank = in->blank;
    p.cs = make_shape(*g);
    p.batch = int(g->batch);
    p.heads = a->heads;
    p.hidden = a->bias_hidden;
    p.inv_patch = float(1.0 / a->patch);
    p.scale = float(1.0 / sqrt(double(a->head_dim)));
}

static int check_inputs(const affmae_attn_inputs* in) {
    if (!in || !in->q || !in->k || !in->v || !in->blank_k || !in->blank_v || !in->coords ||
        !in->w1 || !in->b1 || !in->w2 || !in->b2 || !in->blank)
        return fail(AFFMAE_ECONFIG, "attention: null input pointer");
    return AFFMAE_OK;
}

template <bool BWD>
static int dispatch(const AttnParams& p, int head_dim, int width, cudaStream_t st) {
    const int nt = pick_nt(width), hpc = heads_per_cta(p.heads);
#define AFFMAE_CASE(HD_, NT_, HPC_)                                         \
    if (head_dim == HD_ && nt == NT_ && hpc == HPC_)                        \
        return BWD ? launch_bwd<HD_, NT_, HPC_>(p, st) : launch_fwd<HD_, NT_, HPC_>(p, st);
#define AFFMAE_CASE_NT(HD_, HPC_) AFFMAE_CASE(HD_, 4, HPC_) AFFMAE_CASE(HD_, 7, HPC_)
#define AFFMAE_CASE_HD(HD_) AFFMAE_CASE_NT(HD_, 1) AFFMAE_CASE_NT(HD_, 2) AFFMAE_CASE_NT(HD_, 4)
    AFFMAE_CASE_HD(16)
    AFFMAE_CASE_HD(32)
    AFFMAE_CASE_HD(64)
#undef AFFMAE_CASE_HD
#undef AFFMAE_CASE_NT
#undef AFFMAE_CASE
    return fail(AFFMAE_EUNSUPPORTED, "attention: no compiled kernel variant");
}

static int prepare(AttnParams& p, const AttnWs& w, const int32_t* perm, const int32_t* nbr_cl,
                   const int32_t* rev_cl, int64_t batch, cudaStream_t st) {
    int n = p.heads * kWg2;
    bias_table_kernel<<<(n + 255) / 256, 256, 0, st>>>(p.w1, p.b1, p.w2, p.b2, p.heads, p.hidden, w.tab_g);
    AFFMAE_LAUNCH_CHECK("bias_table_kernel");
    int64_t items = batch * p.cs.c;
    int64_t nk = items * (p.cs.width + 1);
    keylist_kernel<<<unsigned((nk + 255) / 256), 256, 0, st>>>(perm, nbr_cl, p.cs, items, w.keylist);
    AFFMAE_LAUNCH_CHECK("keylist_kernel");
    if (rev_cl) {
        int64_t nq = items * p.cs.g * 16;
        inq_kernel<<<unsigned((nq + 255) / 256), 256, 0, st>>>(perm, rev_cl, p.cs, batch, w.inq);
        AFFMAE_LAUNCH_CHECK("inq_kernel");
    }
    p.tab_g = w.tab_g;
    p.keylist = w.keylist;
    p.inq = w.inq;
    return AFFMAE_OK;
}

size_t attn_fwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (attn_check(g, a)) return 0;
    return carve_ws(g, a, nullptr, false).bytes;
}

size_t attn_bwd_workspace(const affmae_cluster_geom* g, const affmae_attn_desc* a) {
    if (attn_check(g, a)) return 0;
    return carve_ws(g, a, nullptr, true).bytes;
}

int attn_fwd(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
             const int32_t* perm, const int32_t* nbr_cl, affmae_bf16* out, float* lse,
             void* workspace, size_t ws_bytes, void* stream) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if ((rc = check_inputs(in))) return rc;
    if (!perm || !nbr_cl || !out || !lse) return fail(AFFMAE_ECONFIG, "attn_fwd: null pointer");
    AttnWs w = carve_ws(g, a, workspace, false);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "attn_fwd: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    AttnParams p;
    fill_common(p, g, a, in);
    p.perm = perm;
    p.out = reinterpret_cast<__nv_bfloat16*>(out);
    p.lse = lse;
    cudaStream_t st = as_stream(stream);
    if ((rc = prepare(p, w, perm, nbr_cl, nullptr, g->batch, st))) return rc;
    return dispatch<false>(p, a->head_dim, int(g->width), st);
}

int attn_bwd(const affmae_cluster_geom* g, const affmae_attn_desc* a, const affmae_attn_inputs* in,
             const affmae_cluster_index* idx, const affmae_bf16* out, const float* lse,
             const affmae_bf16* dout, affmae_attn_grads* gr, void* workspace, size_t ws_bytes,
             void* stream) {
    int rc = attn_check(g, a);
    if (rc) return rc;
    if ((rc = check_inputs(in))) return rc;
    if (!idx || !idx->perm || !idx->nbr_cl || !idx->rev_off || !idx->rev_cl || !out || !lse ||
        !dout || !gr || !gr->dq || !gr->dk || !gr->dv || !gr->dblank_k || !gr->dblank_v ||
        !gr->dw1 || !gr->db1 || !gr->dw2 || !gr->db2 || !gr->dblank)
        return fail(AFFMAE_ECONFIG, "attn_bwd: null pointer");
    AttnWs w = carve_ws(g, a, workspace, true);
    if (!workspace || ws_bytes < w.bytes) return fail(AFFMAE_ECONFIG, "attn_bwd: workspace too small");
    if (g->batch == 0) return AFFMAE_OK;
    AttnParams p;
    fill_common(p, g, a, in);
    p.perm = idx->perm;
    p.rev_off = idx->rev_off;
    p.out = const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(out));
    p.lse = const_cast<float*>(lse);
    p.dout = reinterpret_cast<const __nv_bfloat16*>(dout);
    p.dq = reinterpret_cast<__nv_bfloat16*>(gr->dq);
    p.dk = reinterpret_cast<__nv_bfloat16*>(gr->dk);
    p.dv = reinterpret_cast<__nv_bfloat16*>(gr->dv);
    p.dsum = w.dsum;
    p.dtab_g = w.dtab_g;
    p.mlp_grad = w.mlp_grad;
    p.blank_grad = w.blank_grad;
    cudaStream_t st = as_stream(stream);
    if ((rc = prepare(p, w, idx->perm, idx->nbr_cl, idx->rev_cl, g->batch, st))) return rc;
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.dtab_g, 0, size_t(a->heads) * kWg2 * 4, st));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.mlp_grad, 0, size_t(a->heads) * (4 * a->bias_hidden + 1) * 4, st));
    AFFMAE_CUDA_CHECK(cudaMemsetAsync(w.blank_grad, 0, size_t(a->heads) * (2 * a->head_dim + 1) * 4, st));
    if ((rc = dispatch<true>(p, a->head_dim, int(g->width), st))) return rc;
    bias_grad_finalize_kernel<<<dim3(16, a->heads), 256, 0, st>>>(w.dtab_g, in->w1, in->b1, in->w2,
                                                                  a->bias_hidden, gr->dw1, gr->db1,
                                                                  gr->dw2, gr->db2);
    AFFMAE_LAUNCH_CHECK("bias_grad_finalize_kernel");
    attn_grad_epilogue_kernel<<<a->heads, 64, 0, st>>>(w.mlp_grad, w.blank_grad, a->heads,
                                                       a->bias_hidden, a->head_dim, gr->dw1,
                                                       gr->db1, gr->dw2, gr->db2, gr->dblank_k,
                                                       gr->dblank_v, gr->dblank);
    AFFMAE_LAUNCH_CHECK("attn_grad_epilogue_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
