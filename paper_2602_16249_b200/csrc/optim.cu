// Fused AdamW over every parameter tensor of the model in one launch
// (AdamW::lr_at / AdamW::step, proj/src/pipeline.cpp:639-680; SURVEY.md §8(f)
// #3): linear warmup then cosine learning rate, bias-corrected moments,
// decoupled weight decay for matrices only (dim(0) > 1).
//
// The parameters live back to back in flat fp32 buffers (value, grad, m, v);
// a device segment table (offsets, decay flags) describes the tensors.  The
// kernel is a persistent grid-stride loop over 4-element vectors: per element
// it reads value, grad, m, v (16 B) and writes value, m, v (12 B) -- HBM-bound,
// 28 algorithmic bytes per parameter.  The schedule and bias corrections are
// scalars of the step (host, binary64); the update runs in fp32 and is stored
// in fp32 (values at the tape precision; the moments are fp32 here, binary64
// in the reference).
#include <cmath>

#include "common.cuh"

namespace affmae_b200 {

struct AdamwScalars {
    double lr, wd, beta1, beta2, bc1, bc2, eps;
};

// decay flag of element `e` (segments sorted by offset; binary search)
__device__ __forceinline__ bool seg_decay_of(const int64_t* __restrict__ off, const uint8_t* __restrict__ decay,
                                             int nseg, int64_t e) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= e) lo = mid;
        else hi = mid - 1;
    }
    return __ldg(decay + lo) != 0;
}

// fp32 arithmetic with the step's scalars folded (1/bc1, 1/bc2 precomputed in binary64);
// the stored values are fp32 either way, so this moves results by ~1 ulp.
struct AdamwF {
    float b1, omb1, b2, omb2, ibc1, ibc2, eps, lr, lrwd;
};
__device__ __forceinline__ float adamw_one(float val, float g, float& m, float& v, bool decay, const AdamwF& s) {
    const float mi = fmaf(s.b1, m, s.omb1 * g);
    const float vi = fmaf(s.b2, v, s.omb2 * g * g);
    m = mi;
    v = vi;
    const float upd = (mi * s.ibc1) / (sqrtf(vi * s.ibc2) + s.eps);
    float x = val;
    if (decay) x = fmaf(-s.lrwd, x, x);
    return fmaf(-s.lr, upd, x);
}

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ value, const float* __restrict__ grad,
                                                    float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                    const int64_t* __restrict__ off, const uint8_t* __restrict__ decay,
                                                    int nseg, AdamwF s) {
    const int64_t nv = n / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const int64_t e = 4 * i;
        // a 4-vector may straddle a segment boundary: flags per element
        const bool d0 = seg_decay_of(off, decay, nseg, e), d3 = seg_decay_of(off, decay, nseg, e + 3);
        float4 x = reinterpret_cast<float4*>(value)[i];
        const float4 g = __ldg(reinterpret_cast<const float4*>(grad) + i);
        float4 mm = reinterpret_cast<float4*>(m)[i], vv = reinterpret_cast<float4*>(v)[i];
        bool dd[4] = {d0, d0, d0, d3};
        if (d0 != d3) {
            dd[1] = seg_decay_of(off, decay, nseg, e + 1);
            dd[2] = seg_decay_of(off, decay, nseg, e + 2);
        }
        x.x = adamw_one(x.x, g.x, mm.x, vv.x, dd[0], s);
        x.y = adamw_one(x.y, g.y, mm.y, vv.y, dd[1], s);
        x.z = adamw_one(x.z, g.z, mm.z, vv.z, dd[2], s);
        x.w = adamw_one(x.w, g.w, mm.w, vv.w, dd[3], s);
        reinterpret_cast<float4*>(value)[i] = x;
        reinterpret_cast<float4*>(m)[i] = mm;
        reinterpret_cast<float4*>(v)[i] = vv;
    }
    // tail (n % 4 elements)
    const int64_t t = 4 * nv + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n) {
        float mm = m[t], vv = v[t];
        value[t] = adamw_one(value[t], grad[t], mm, vv, seg_decay_of(off, decay, nseg, t), s);
        m[t] = mm;
        v[t] = vv;
    }
}

// ---- step-count-on-device variant (the training step's CUDA graph replays it unchanged):
// a one-thread prologue derives the step's scalars from *step (AdamW::t_) in binary64 and
// advances it; the update kernel also refreshes the bf16 shadow of the first n_shadow
// values (the tensor-core operands of the model's GEMMs).
__global__ void adamw_scalars_kernel(affmae_adamw_cfg c, int64_t* __restrict__ step, AdamwF* __restrict__ out) {
    const int64_t t = *step;
    double lr;
    if (t < c.warmup) {
        lr = c.lr * double(t + 1) / double(c.warmup);
    } else {
        const int64_t span = c.total_steps - c.warmup > 1 ? c.total_steps - c.warmup : 1;
        double prog = double(t - c.warmup) / double(span);
        prog = prog < 1.0 ? prog : 1.0;
        lr = c.lr * 0.5 * (1.0 + cos(3.14159265358979323846 * prog));
    }
    const double nn = double(t + 1);
    AdamwF f;
    f.b1 = float(c.beta1);
    f.omb1 = float(1.0 - c.beta1);
    f.b2 = float(c.beta2);
    f.omb2 = float(1.0 - c.beta2);
    f.ibc1 = float(1.0 / (1.0 - pow(c.beta1, nn)));
    f.ibc2 = float(1.0 / (1.0 - pow(c.beta2, nn)));
    f.eps = 1e-8f;
    f.lr = float(lr);
    f.lrwd = float(lr * c.weight_decay);
    *out = f;
    *step = t + 1;
}

__global__ void __launch_bounds__(256) adamw_dev_kernel(float* __restrict__ value, const float* __restrict__ grad,
                                                        float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                        const int64_t* __restrict__ off,
                                                        const uint8_t* __restrict__ decay, int nseg,
                                                        const AdamwF* __restrict__ sp, __nv_bfloat16* __restrict__ shadow,
                                                        int64_t n_shadow) {
    const AdamwF s = *sp;
    const int64_t nv = n / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const int64_t e = 4 * i;
        const bool d0 = seg_decay_of(off, decay, nseg, e), d3 = seg_decay_of(off, decay, nseg, e + 3);
        float4 x = reinterpret_cast<float4*>(value)[i];
        const float4 g = __ldg(reinterpret_cast<const float4*>(grad) + i);
        float4 mm = reinterpret_cast<float4*>(m)[i], vv = reinterpret_cast<float4*>(v)[i];
        bool dd[4] = {d0, d0, d0, d3};
        if (d0 != d3) {
            dd[1] = seg_decay_of(off, decay, nseg, e + 1);
            dd[2] = seg_decay_of(off, decay, nseg, e + 2);
        }
        x.x = adamw_one(x.x, g.x, mm.x, vv.x, dd[0], s);
        x.y = adamw_one(x.y, g.y, mm.y, vv.y, dd[1], s);
        x.z = adamw_one(x.z, g.z, mm.z, vv.z, dd[2], s);
        x.w = adamw_one(x.w, g.w, mm.w, vv.w, dd[3], s);
        reinterpret_cast<float4*>(value)[i] = x;
        reinterpret_cast<float4*>(m)[i] = mm;
        reinterpret_cast<float4*>(v)[i] = vv;
        if (e < n_shadow) {
            __nv_bfloat162 h[2] = {__floats2bfloat162_rn(x.x, x.y), __floats2bfloat162_rn(x.z, x.w)};
            *reinterpret_cast<uint2*>(shadow + e) = *reinterpret_cast<const uint2*>(h);
        }
    }
}

int adamw_step_dev(const affmae_adamw_cfg* c, int64_t* step_dev, void* scalars_dev, int64_t n_segments,
                   const int64_t* seg_off, const uint8_t* seg_decay, int64_t n, float* value, const float* grad,
                   float* m, float* v, void* shadow, int64_t n_shadow, void* stream) {
    if (!c || !step_dev || !scalars_dev || !seg_off || !seg_decay || !value || !grad || !m || !v)
        return fail(AFFMAE_ECONFIG, "adamw: null pointer");
    if (c->total_steps < 1) return fail(AFFMAE_ECONFIG, "optimizer needs at least one step");
    if (n % 4 || n_shadow % 4 || n_shadow > n || (n_shadow && !shadow))
        return fail(AFFMAE_ECONFIG, "adamw: sizes must be multiples of 4");
    cudaStream_t st = as_stream(stream);
    adamw_scalars_kernel<<<1, 1, 0, st>>>(*c, step_dev, static_cast<AdamwF*>(scalars_dev));
    const int64_t work = n / 4;
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8 * kNumSMs)));
    adamw_dev_kernel<<<blocks, 256, 0, st>>>(value, grad, m, v, n, seg_off, seg_decay, int(n_segments),
                                             static_cast<const AdamwF*>(scalars_dev),
                                             static_cast<__nv_bfloat16*>(shadow), n_shadow);
    AFFMAE_LAUNCH_CHECK("adamw_dev_kernel");
    return AFFMAE_OK;
}
size_t adamw_scalars_bytes() { return sizeof(AdamwF); }

double adamw_lr(const affmae_adamw_cfg* c, int64_t step) {
    if (step < c->warmup) return c->lr * double(step + 1) / double(c->warmup);
    const int64_t span = c->total_steps - c->warmup > 1 ? c->total_steps - c->warmup : 1;
    double prog = double(step - c->warmup) / double(span);
    prog = prog < 1.0 ? prog : 1.0;
    return c->lr * 0.5 * (1.0 + std::cos(3.14159265358979323846 * prog));
}

int adamw_step(const affmae_adamw_cfg* c, int64_t step, int64_t n_segments, const int64_t* seg_off,
               const uint8_t* seg_decay, int64_t n, float* value, const float* grad, float* m, float* v,
               void* stream) {
    if (!c || !seg_off || !seg_decay || !value || !grad || !m || !v)
        return fail(AFFMAE_ECONFIG, "adamw: null pointer");
    if (c->total_steps < 1) return fail(AFFMAE_ECONFIG, "optimizer needs at least one step");
    if (step < 0 || n_segments < 1 || n < 0) return fail(AFFMAE_ECONFIG, "adamw: bad step / sizes");
    if (n_segments > (int64_t(1) << 30)) return fail(AFFMAE_EUNSUPPORTED, "adamw: too many segments");
    if ((reinterpret_cast<uintptr_t>(value) | reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(m) |
         reinterpret_cast<uintptr_t>(v)) & 15)
        return fail(AFFMAE_ECONFIG, "adamw: buffers must be 16-byte aligned");
    if (n == 0) return AFFMAE_OK;
    AdamwScalars s;
    const double nn = double(step + 1);
    s.lr = adamw_lr(c, step);
    s.wd = c->weight_decay;
    s.beta1 = c->beta1;
    s.beta2 = c->beta2;
    s.bc1 = 1.0 - std::pow(c->beta1, nn);
    s.bc2 = 1.0 - std::pow(c->beta2, nn);
    s.eps = 1e-8;  // kAdamEps, pipeline.cpp:24
    AdamwF f;
    f.b1 = float(s.beta1);
    f.omb1 = float(1.0 - s.beta1);
    f.b2 = float(s.beta2);
    f.omb2 = float(1.0 - s.beta2);
    f.ibc1 = float(1.0 / s.bc1);
    f.ibc2 = float(1.0 / s.bc2);
    f.eps = float(s.eps);
    f.lr = float(s.lr);
    f.lrwd = float(s.lr * s.wd);
    const int64_t work = (n + 3) / 4;
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8 * kNumSMs)));
    adamw_kernel<<<blocks, 256, 0, as_stream(stream)>>>(value, grad, m, v, n, seg_off, seg_decay, int(n_segments),
                                                        f);
    AFFMAE_LAUNCH_CHECK("adamw_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
