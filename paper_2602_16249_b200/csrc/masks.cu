// Device-side Perlin patch masks and stage-0 coordinates:
// perlin_field + mask_from_field (proj/src/masking.cpp:34-92) and the visible
// patch-centre lattice (proj/src/geometry.cpp:44-50, proj/src/pipeline.cpp:412-427),
// batched over images so a training step needs no host-side mask work.
//
// Bit-exact with the reference: the corner gradients need cos / sin of the hashed
// angle, whose correctly rounded host values (glibc) the device libm does not
// guarantee, so the host computes the few gradients a grid touches ((freq+1)^2 per
// octave) and the device evaluates the field with explicitly rounded binary64 ops
// (__dmul_rn / __dadd_rn: no FMA contraction), in the reference's operation order.
// Selection: exactly round(ratio * cells) cells, largest field value first, ties to
// the lower cell index -- a per-image 8-pass radix select over the order-preserving
// 64-bit image of the doubles, then the equal-to-threshold cells ranked by index
// with a block scan.  One 1024-thread block per image.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace affmae_b200 {

constexpr int kMaskThreads = 1024;

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double fade_rn(double t) {
    // t * t * t * (t * (t * 6.0 - 15.0) + 10.0), left to right
    const double t3 = dm(dm(t, t), t);
    return dm(t3, da(dm(t, ds(dm(t, 6.0), 15.0)), 10.0));
}
__device__ __forceinline__ double lerp_rn(double a, double b, double t) { return da(a, dm(ds(b, a), t)); }

// grads: per image, per octave, (side x side) corners {gx, gy}, side = freq + 1 (+1 spare)
struct PerlinGeo {
    int64_t h, w;
    int octaves;
    double base_freq;
    int64_t corners;  // per image, all octaves
};

__global__ void perlin_field_kernel(const double2* __restrict__ grads, const int64_t* __restrict__ oct_off,
                                    const int32_t* __restrict__ oct_side, const double* __restrict__ amp,
                                    PerlinGeo g, int64_t batch, double* __restrict__ field) {
    const int64_t cells = g.h * g.w, n = batch * cells;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / cells, c = t - b * cells, i = c / g.w, j = c - i * g.w;
        const double2* gb = grads + b * g.corners;
        double acc = 0.0;
        for (int o = 0; o < g.octaves; ++o) {
            const double freq = g.base_freq * double(1 << o);
            const double py = __ddiv_rn(dm(double(i), freq), double(g.h));
            const double px = __ddiv_rn(dm(double(j), freq), double(g.w));
            const double fx0 = floor(px), fy0 = floor(py);
            const int x0 = int(fx0), y0 = int(fy0), side = oct_side[o];
            const double tx = ds(px, fx0), ty = ds(py, fy0);
            const double2* go = gb + oct_off[o];
            const double2 g00 = go[y0 * side + x0], g10 = go[y0 * side + x0 + 1];
            const double2 g01 = go[(y0 + 1) * side + x0], g11 = go[(y0 + 1) * side + x0 + 1];
            const double n00 = da(dm(g00.x, tx), dm(g00.y, ty));
            const double n10 = da(dm(g10.x, ds(tx, 1.0)), dm(g10.y, ty));
            const double n01 = da(dm(g01.x, tx), dm(g01.y, ds(ty, 1.0)));
            const double n11 = da(dm(g11.x, ds(tx, 1.0)), dm(g11.y, ds(ty, 1.0)));
            const double u = fade_rn(tx), v = fade_rn(ty);
            const double val = lerp_rn(lerp_rn(n00, n10, u), lerp_rn(n01, n11, u), v);
            acc = da(acc, dm(amp[o], val));
        }
        field[t] = acc;
    }
}

// order-preserving image of a double, complemented so that larger values get smaller keys
__device__ __forceinline__ uint64_t desc_key(double v) {
    uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
    u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    return ~u;
}

__global__ void __launch_bounds__(kMaskThreads) mask_select_kernel(const double* __restrict__ field, int64_t cells,
                                                                   int64_t want, uint8_t* __restrict__ masked) {
    constexpr int kCand = 4096;  // candidates kept in shared memory once they fit
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_rank;
    __shared__ int32_t wsum[32];
    __shared__ uint64_t cand[kCand];
    __shared__ int32_t s_ncand, s_cnt;
    __shared__ bool s_use;
    const double* f = field + int64_t(blockIdx.x) * cells;
    uint8_t* m = masked + int64_t(blockIdx.x) * cells;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_rank = want;  // 1-based rank of the threshold among the keys matching the prefix
        s_ncand = 0;
        s_use = false;
    }
    __syncthreads();
    if (want <= 0) {
        for (int64_t i = threadIdx.x; i < cells; i += kMaskThreads) m[i] = 0;
        return;
    }
    // radix select (ascending keys = descending values) of the want-th smallest key
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
        for (int i = threadIdx.x; i < 256; i += kMaskThreads) hist[i] = 0;
        __syncthreads();
        const uint64_t pre = s_prefix;
        if (s_use) {
            for (int i = threadIdx.x; i < s_ncand; i += kMaskThreads) {
                const uint64_t k = cand[i];
                if ((k & hi_mask) == pre) atomicAdd(&hist[(k >> shift) & 255], 1u);
            }
        } else {
            for (int64_t i = threadIdx.x; i < cells; i += kMaskThreads) {
                const uint64_t k = desc_key(f[i]);
                if ((k & hi_mask) == pre) atomicAdd(&hist[(k >> shift) & 255], 1u);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t r = s_rank;
            int d = 0;
            for (; d < 256; ++d) {
                if (r <= int64_t(hist[d])) break;
                r -= hist[d];
            }
            s_prefix = pre | (uint64_t(d) << shift);
            s_rank = r;
            s_cnt = int32_t(hist[d < 256 ? d : 255]);
        }
        __syncthreads();
        // once the keys under the new prefix fit, keep only them (later passes stop re-reading)
        if (!s_use && s_cnt <= kCand && pass < 7) {
            const uint64_t npre = s_prefix, nmask = ~0ull << shift;
            for (int64_t i = threadIdx.x; i < cells; i += kMaskThreads) {
                const uint64_t k = desc_key(f[i]);
                if ((k & nmask) == npre) cand[atomicAdd(&s_ncand, 1)] = k;
            }
            __syncthreads();
            if (threadIdx.x == 0) s_use = true;
            __syncthreads();
        }
    }
    const uint64_t T = s_prefix;
    const int64_t take_eq = s_rank;  // equal-to-T cells to take, lowest index first
    // rank the equal cells by index: contiguous chunks per thread + block scan
    const int64_t per = (cells + kMaskThreads - 1) / kMaskThreads;
    const int64_t lo = threadIdx.x * per, hi = lo + per < cells ? lo + per : cells;
    int32_t eq = 0;
    for (int64_t i = lo; i < hi; ++i) eq += desc_key(f[i]) == T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t inc = eq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    int64_t before = inc - eq + (warp > 0 ? wsum[warp - 1] : 0);
    for (int64_t i = lo; i < hi; ++i) {
        const uint64_t k = desc_key(f[i]);
        uint8_t out = k < T;
        if (k == T) out = before++ < take_eq;
        m[i] = out;
    }
}

// visible cells' pixel centres in ascending cell index: per-image block scan
__global__ void __launch_bounds__(kMaskThreads) visible_coords_kernel(const uint8_t* __restrict__ masked, int64_t h,
                                                                      int64_t w, double patch, int64_t nvis,
                                                                      float2* __restrict__ coords,
                                                                      int32_t* __restrict__ count) {
    __shared__ int32_t wsum[32];
    const int64_t cells = h * w;
    const uint8_t* m = masked + int64_t(blockIdx.x) * cells;
    float2* out = coords + int64_t(blockIdx.x) * nvis;
    const int64_t per = (cells + kMaskThreads - 1) / kMaskThreads;
    const int64_t lo = threadIdx.x * per, hi = lo + per < cells ? lo + per : cells;
    int32_t vis = 0;
    for (int64_t i = lo; i < hi; ++i) vis += m[i] == 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t inc = vis;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    int64_t pos = inc - vis + (warp > 0 ? wsum[warp - 1] : 0);
    for (int64_t i = lo; i < hi; ++i)
        if (m[i] == 0) {
            if (pos < nvis) {
                const int64_t r = i / w, c = i - r * w;
                out[pos] = make_float2(float(double(c) * patch + patch * 0.5), float(double(r) * patch + patch * 0.5));
            }
            ++pos;
        }
    if (threadIdx.x == kMaskThreads - 1 && count) count[blockIdx.x] = wsum[31];
}

static uint64_t mix64_h(uint64_t z) {  // proj/include/affmae/rng.hpp:8-13
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

size_t perlin_mask_workspace(int64_t batch, int64_t h, int64_t w, int octaves, double base_freq) {
    int64_t corners = 0;
    for (int o = 0; o < octaves; ++o) {
        const int64_t side = int64_t(std::ceil(base_freq * double(1 << o))) + 2;
        corners += side * side;
    }
    return ((size_t(batch * h * w) * 8 + 255) & ~size_t(255)) + size_t(batch * corners) * 16 + size_t(octaves) * 32 +
           1024;
}

// The Perlin field of `batch` images into the start of `workspace` (perlin_mask_workspace
// layout): host gradient table + amplitudes, uploaded on `st`, then perlin_field_kernel.
static int perlin_field_only(const uint64_t* seeds, int64_t batch, int64_t h, int64_t w, int octaves,
                             double base_freq, double persistence, void* workspace, cudaStream_t st) {
    // host: the corner gradients a grid touches (proj/src/masking.cpp:21-26, 51-69)
    const size_t no = static_cast<size_t>(octaves);
    std::vector<int64_t> off(no);
    std::vector<int32_t> side(no);
    std::vector<double> amp(no);
    int64_t corners = 0;
    for (int o = 0; o < octaves; ++o) {
        side[size_t(o)] = int32_t(std::ceil(base_freq * double(1 << o))) + 2;
        off[size_t(o)] = corners;
        corners += int64_t(side[size_t(o)]) * side[size_t(o)];
        amp[size_t(o)] = std::pow(persistence, o);
    }
    std::vector<double> grads(static_cast<size_t>(batch * corners) * 2);
    for (int64_t b = 0; b < batch; ++b)
        for (int o = 0; o < octaves; ++o) {
            const uint64_t os = mix64_h(seeds[b] + 0x9E3779B97F4A7C15ull * uint64_t(o + 1));
            const int s = side[size_t(o)];
            for (int iy = 0; iy < s; ++iy)
                for (int ix = 0; ix < s; ++ix) {
                    const uint64_t k = mix64_h(mix64_h(uint64_t(ix) * 0x9E3779B97F4A7C15ull ^ uint64_t(iy)) ^ os);
                    const double ang = double(k >> 11) * 0x1.0p-53 * 6.283185307179586476925287;
                    const size_t e = size_t(b * corners + off[size_t(o)] + iy * s + ix) * 2;
                    grads[e] = std::cos(ang);
                    grads[e + 1] = std::sin(ang);
                }
        }
    char* ws = static_cast<char*>(workspace);
    double* field = reinterpret_cast<double*>(ws);
    double2* dgr = reinterpret_cast<double2*>(ws + ((size_t(batch * h * w) * 8 + 255) & ~size_t(255)));
    char* meta = reinterpret_cast<char*>(dgr + batch * corners);
    int64_t* doff = reinterpret_cast<int64_t*>(meta);
    double* damp = reinterpret_cast<double*>(doff + octaves);
    int32_t* dside = reinterpret_cast<int32_t*>(damp + octaves);
    // pageable copies are staged by the driver before returning: the host vectors may die
    if (cudaMemcpyAsync(dgr, grads.data(), grads.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(doff, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(damp, amp.data(), amp.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(dside, side.data(), side.size() * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return fail(AFFMAE_ECUDA, "perlin_field: H2D of the gradient table failed");
    PerlinGeo g{h, w, octaves, base_freq, corners};
    const int64_t n = batch * h * w;
    perlin_field_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 16 * kNumSMs)), 256, 0, st>>>(
        dgr, doff, dside, damp, g, batch, field);
    AFFMAE_LAUNCH_CHECK("perlin_field_kernel");
    return AFFMAE_OK;
}

int perlin_mask(const uint64_t* seeds, int64_t batch, int64_t h, int64_t w, int octaves, double base_freq,
                double persistence, double ratio, uint8_t* masked, void* workspace, size_t ws_bytes, void* stream) {
    if (!seeds || !masked) return fail(AFFMAE_ECONFIG, "perlin_mask: null pointer");
    if (h < 2 || w < 2) return fail(AFFMAE_ECONFIG, "perlin_field: grid must be at least 2x2");
    if (octaves < 1 || octaves > 16) return fail(AFFMAE_ECONFIG, "perlin_field: octaves must be in [1, 16]");
    if (!(ratio >= 0.0 && ratio <= 1.0)) return fail(AFFMAE_ECONFIG, "mask_from_field: ratio must be in [0, 1]");
    if (!(base_freq > 0.0)) return fail(AFFMAE_ECONFIG, "perlin_field: base_freq must be positive");
    if (batch < 0) return fail(AFFMAE_ECONFIG, "perlin_mask: bad batch");
    if (!workspace || ws_bytes < perlin_mask_workspace(batch, h, w, octaves, base_freq))
        return fail(AFFMAE_ECONFIG, "perlin_mask: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    int rc = perlin_field_only(seeds, batch, h, w, octaves, base_freq, persistence, workspace, st);
    if (rc) return rc;
    const int64_t want = std::llround(ratio * double(h * w));
    mask_select_kernel<<<unsigned(batch), kMaskThreads, 0, st>>>(static_cast<const double*>(workspace), h * w, want,
                                                                 masked);
    AFFMAE_LAUNCH_CHECK("perlin_mask");
    return AFFMAE_OK;
}

int visible_coords(const uint8_t* masked, int64_t batch, int64_t h, int64_t w, double patch, int64_t nvis,
                   float* coords, int32_t* count, void* stream) {
    if (!masked || !coords) return fail(AFFMAE_ECONFIG, "visible_coords: null pointer");
    if (batch < 0 || h < 1 || w < 1 || nvis < 0) return fail(AFFMAE_ECONFIG, "visible_coords: bad shape");
    if (batch == 0) return AFFMAE_OK;
    visible_coords_kernel<<<unsigned(batch), kMaskThreads, 0, as_stream(stream)>>>(
        masked, h, w, patch, nvis, reinterpret_cast<float2*>(coords), count);
    AFFMAE_LAUNCH_CHECK("visible_coords_kernel");
    return AFFMAE_OK;
}

// ---------------------------------------------------------------------------
// synth_image (proj/src/pipeline.cpp:169-227) on the device, batched: the Perlin base
// (perlin_field(size, size, 2, 2.0, 0.5, mix64(seed ^ 0xba5e11)) through the same host
// gradient table + explicitly rounded field kernel as the masks), then per curve the
// max-of-stamps ink buffer (the stamps scatter with a 64-bit atomic max on the bit
// pattern: the weights are positive, so the order of the doubles is the order of their
// bits) added in curve order, the Gaussian blobs, and the clamp.  The RNG draws (splitmix64
// stream, include/affmae/rng.hpp) stay on the host: a few dozen numbers per image.  exp()
// is the device libm (<= 1 ulp from glibc), so pixels match the reference to ~1e-15, not
// bitwise.
namespace {
struct HostRng {  // include/affmae/rng.hpp:18-44
    uint64_t s;
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t below(uint64_t n) { return n ? next() % n : 0; }
};
}  // namespace

constexpr int kSynthMaxCurves = 4, kSynthMaxBlobs = 5;

struct SynthParams {          // per image
    int curves, blobs;
    double cpx[kSynthMaxCurves][3], cpy[kSynthMaxCurves][3], csig[kSynthMaxCurves], camp[kSynthMaxCurves];
    double bx[kSynthMaxBlobs], by[kSynthMaxBlobs], bsig[kSynthMaxBlobs], bamp[kSynthMaxBlobs];
};

__global__ void synth_base_kernel(const double* __restrict__ field, int64_t n, double* __restrict__ img) {
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x)
        img[t] = da(0.5, dm(0.3, field[t]));
}

// one thread per (image, step, box cell); box side <= 2*ceil(3*sigma)+2 <= 14 for sigma < 1.8
constexpr int kStampSide = 16;
__global__ void synth_stamp_kernel(const SynthParams* __restrict__ prm, int c, int64_t size, int64_t batch,
                                   unsigned long long* __restrict__ ink) {
    const int64_t nsteps = 3 * size, per_img = (nsteps + 1) * kStampSide * kStampSide;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < batch * per_img;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / per_img, rem = t - b * per_img, st = rem / (kStampSide * kStampSide);
        const int cell = int(rem - st * kStampSide * kStampSide), rr = cell / kStampSide, cc0 = cell % kStampSide;
        const SynthParams& P = prm[b];
        if (c >= P.curves) continue;
        const double u = __ddiv_rn(double(st), double(nsteps));
        const double a = dm(ds(1.0, u), ds(1.0, u)), bq = dm(dm(2.0, u), ds(1.0, u)), c2 = dm(u, u);
        const double cx = da(da(dm(a, P.cpx[c][0]), dm(bq, P.cpx[c][1])), dm(c2, P.cpx[c][2]));
        const double cy = da(da(dm(a, P.cpy[c][0]), dm(bq, P.cpy[c][1])), dm(c2, P.cpy[c][2]));
        const double sg = P.csig[c], s3 = dm(3.0, sg);
        const int64_t r0 = max(int64_t(0), int64_t(floor(ds(cy, s3))));
        const int64_t r1 = min(size - 1, int64_t(ceil(da(cy, s3))));
        const int64_t c0 = max(int64_t(0), int64_t(floor(ds(cx, s3))));
        const int64_t c1 = min(size - 1, int64_t(ceil(da(cx, s3))));
        const int64_t r = r0 + rr, col = c0 + cc0;
        if (r > r1 || col > c1) continue;
        const double dx = ds(da(double(col), 0.5), cx), dy = ds(da(double(r), 0.5), cy);
        const double wgt = exp(__ddiv_rn(-da(dm(dx, dx), dm(dy, dy)), dm(dm(2.0, sg), sg)));
        if (wgt > 0.0) atomicMax(ink + b * size * size + r * size + col, (unsigned long long)__double_as_longlong(wgt));
    }
}

__global__ void synth_ink_add_kernel(const SynthParams* __restrict__ prm, int c, int64_t size, int64_t batch,
                                     unsigned long long* __restrict__ ink, double* __restrict__ img) {
    const int64_t cells = size * size;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < batch * cells;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / cells;
        if (c < prm[b].curves) img[t] = da(img[t], dm(prm[b].camp[c], __longlong_as_double((long long)ink[t])));
        ink[t] = 0ull;
    }
}

__global__ void synth_blobs_kernel(const SynthParams* __restrict__ prm, int64_t size, int64_t batch,
                                   double* __restrict__ img) {
    const int64_t cells = size * size;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < batch * cells;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / cells, i = t - b * cells, r = i / size, c = i - r * size;
        const SynthParams& P = prm[b];
        double v = img[t];
        for (int k = 0; k < P.blobs; ++k) {
            const double dx = ds(da(double(c), 0.5), P.bx[k]), dy = ds(da(double(r), 0.5), P.by[k]);
            v = da(v, dm(P.bamp[k], exp(__ddiv_rn(-da(dm(dx, dx), dm(dy, dy)), dm(dm(2.0, P.bsig[k]), P.bsig[k])))));
        }
        img[t] = fmin(fmax(v, 0.0), 1.0);
    }
}

size_t synth_images_workspace(int64_t batch, int64_t size) {
    return perlin_mask_workspace(batch, size, size, 2, 2.0) + size_t(batch * size * size) * 8 +
           size_t(batch) * sizeof(SynthParams) + 1280;
}

int synth_images(const uint64_t* seeds, int64_t batch, int64_t size, double* img, void* workspace, size_t ws_bytes,
                 void* stream) {
    if (!seeds || !img) return fail(AFFMAE_ECONFIG, "synth_image: null pointer");
    if (size < 2) return fail(AFFMAE_ECONFIG, "synth_image: size must be >= 2");
    if (batch < 0) return fail(AFFMAE_ECONFIG, "synth_image: bad batch");
    if (!workspace || ws_bytes < synth_images_workspace(batch, size))
        return fail(AFFMAE_ECONFIG, "synth_image: workspace too small");
    if (batch == 0) return AFFMAE_OK;
    cudaStream_t st = as_stream(stream);
    std::vector<uint64_t> fseeds(static_cast<size_t>(batch));
    std::vector<SynthParams> prm(static_cast<size_t>(batch));
    for (int64_t b = 0; b < batch; ++b) {
        fseeds[size_t(b)] = mix64_h(seeds[b] ^ 0xba5e11ull);
        HostRng rng{mix64_h(seeds[b]) ^ 0x5ca1ab1eull};
        SynthParams& P = prm[size_t(b)];
        P.curves = 2 + int(rng.below(3));
        for (int c = 0; c < P.curves; ++c) {
            for (int j = 0; j < 3; ++j) {
                P.cpx[c][j] = rng.uniform(0.0, double(size));
                P.cpy[c][j] = rng.uniform(0.0, double(size));
            }
            P.csig[c] = rng.uniform(0.8, 1.8);
            P.camp[c] = rng.uniform(0.25, 0.45) * (rng.below(2) ? 1.0 : -1.0);
        }
        P.blobs = 2 + int(rng.below(4));
        for (int k = 0; k < P.blobs; ++k) {
            P.bx[k] = rng.uniform(0.0, double(size));
            P.by[k] = rng.uniform(0.0, double(size));
            P.bsig[k] = rng.uniform(2.0, std::max(3.0, double(size) / 8.0));
            P.bamp[k] = rng.uniform(0.3, 0.5) * (rng.below(2) ? 1.0 : -1.0);
        }
    }
    char* ws = static_cast<char*>(workspace);
    const size_t pws = perlin_mask_workspace(batch, size, size, 2, 2.0);
    auto* ink = reinterpret_cast<unsigned long long*>(ws + ((pws + 255) & ~size_t(255)));
    auto* dprm = reinterpret_cast<SynthParams*>(ink + batch * size * size);
    // the Perlin field of perlin_mask's pipeline, without the selection (field at ws start)
    int rc = perlin_field_only(fseeds.data(), batch, size, size, 2, 2.0, 0.5, ws, st);
    if (rc) return rc;
    if (cudaMemcpyAsync(dprm, prm.data(), prm.size() * sizeof(SynthParams), cudaMemcpyHostToDevice, st) !=
            cudaSuccess ||
        cudaMemsetAsync(ink, 0, size_t(batch * size * size) * 8, st) != cudaSuccess)
        return fail(AFFMAE_ECUDA, "synth_image: staging failed");
    const int64_t n = batch * size * size;
    const unsigned nb = unsigned(std::min<int64_t>((n + 255) / 256, 16 * kNumSMs));
    synth_base_kernel<<<nb, 256, 0, st>>>(reinterpret_cast<const double*>(ws), n, img);
    const int64_t stamps = batch * (3 * size + 1) * kStampSide * kStampSide;
    const unsigned sb = unsigned(std::min<int64_t>((stamps + 255) / 256, 32 * kNumSMs));
    for (int c = 0; c < kSynthMaxCurves; ++c) {
        synth_stamp_kernel<<<sb, 256, 0, st>>>(dprm, c, size, batch, ink);
        synth_ink_add_kernel<<<nb, 256, 0, st>>>(dprm, c, size, batch, ink, img);
    }
    synth_blobs_kernel<<<nb, 256, 0, st>>>(dprm, size, batch, img);
    AFFMAE_LAUNCH_CHECK("synth_images");
    // the host staging vectors must outlive the async copies
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(AFFMAE_ECUDA, "synth_image: sync failed");
    return AFFMAE_OK;
}

// ---------------------------------------------------------------------------
// patchify (proj/src/pipeline.cpp:131-150) and the masked-cell target rows of the loss
// (Model::loss_parts, :588-596): image [B, H, W] float64 -> vectors [B, T, patch^2] float32
// (the b32 tape's rounding of Tensor::set), and the masked cells of every image in
// ascending index as GLOBAL rows b*T + cell (what affmae_masked_mse gathers).
__global__ void patchify_kernel(const double* __restrict__ img, int64_t batch, int64_t h, int64_t w, int patch,
                                float* __restrict__ vec) {
    const int64_t gw = w / patch, cells = (h / patch) * gw, p2 = int64_t(patch) * patch, per = cells * p2;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < batch * per;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t / per, r = t - b * per, tix = r / p2, e = r - tix * p2;
        const int64_t gr = tix / gw, gc = tix - gr * gw, pr = e / patch, pc = e - pr * patch;
        vec[t] = float(img[(b * h + gr * patch + pr) * w + gc * patch + pc]);
    }
}

__global__ void __launch_bounds__(kMaskThreads) masked_rows_kernel(const uint8_t* __restrict__ masked, int64_t cells,
                                                                   int64_t nmask, int32_t* __restrict__ rows) {
    __shared__ int32_t wsum[32];
    const uint8_t* m = masked + int64_t(blockIdx.x) * cells;
    int32_t* out = rows + int64_t(blockIdx.x) * nmask;
    const int64_t per = (cells + kMaskThreads - 1) / kMaskThreads;
    const int64_t lo = threadIdx.x * per, hi = lo + per < cells ? lo + per : cells;
    int32_t cnt = 0;
    for (int64_t i = lo; i < hi; ++i) cnt += m[i] != 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += v;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    int64_t pos = inc - cnt + (warp > 0 ? wsum[warp - 1] : 0);
    for (int64_t i = lo; i < hi; ++i)
        if (m[i] != 0) {
            if (pos < nmask) out[pos] = int32_t(int64_t(blockIdx.x) * cells + i);
            ++pos;
        }
}

int patchify(const double* img, int64_t batch, int64_t h, int64_t w, int64_t patch, float* vectors, void* stream) {
    if (!img || !vectors) return fail(AFFMAE_ECONFIG, "patchify: null pointer");
    if (patch < 1 || h % patch || w % patch || h < patch || w < patch)
        return fail(AFFMAE_ECONFIG, "patchify: image extents must be positive multiples of the patch");
    if (batch <= 0) return batch == 0 ? AFFMAE_OK : fail(AFFMAE_ECONFIG, "patchify: bad batch");
    const int64_t n = batch * h * w;
    patchify_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 16 * kNumSMs)), 256, 0, as_stream(stream)>>>(
        img, batch, h, w, int(patch), vectors);
    AFFMAE_LAUNCH_CHECK("patchify_kernel");
    return AFFMAE_OK;
}

int masked_rows(const uint8_t* masked, int64_t batch, int64_t cells, int64_t nmask, int32_t* rows, void* stream) {
    if (!masked || !rows) return fail(AFFMAE_ECONFIG, "masked_rows: null pointer");
    if (batch < 0 || cells < 1 || nmask < 0 || batch * cells >= (int64_t(1) << 31))
        return fail(AFFMAE_ECONFIG, "masked_rows: bad shape");
    if (batch == 0) return AFFMAE_OK;
    masked_rows_kernel<<<unsigned(batch), kMaskThreads, 0, as_stream(stream)>>>(masked, cells, nmask, rows);
    AFFMAE_LAUNCH_CHECK("masked_rows_kernel");
    return AFFMAE_OK;
}

}  // namespace affmae_b200
