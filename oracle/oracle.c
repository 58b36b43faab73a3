/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 *
 * This file is the parity checker (see oracle.h).  It is never linked into
 * the product library and never on a measured path except bench.py's
 * cpu_baseline leg.  Parity of this restatement is PINNED: the CPU test suite
 * compares it bit-for-bit against the reference compiled unmodified
 * (oracle/_ref, built from /root/reference/proj/src) and against the golden
 * vectors in tests/golden/ that the reference produced.
 *
 * Arithmetic follows the reference's evaluation order exactly, with FP
 * contraction disabled (-ffp-contract=off), matching the reference's
 * x86-64 build (no FMA, no -ffast-math: proj/CMakeLists.txt:13-14).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NEG_INF (-INFINITY)

/* ------------------------------------------------------------------ sorting */

typedef struct {
    uint64_t key;
    int64_t idx;
} KeyIdx;

static int cmp_keyidx(const void* a, const void* b) {
    const KeyIdx* x = (const KeyIdx*)a;
    const KeyIdx* y = (const KeyIdx*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

typedef struct {
    double d;
    int64_t idx;
} DistIdx;

/* std::pair<double, int64_t> ordering */
static int pair_less(DistIdx a, DistIdx b) { return a.d < b.d || (!(b.d < a.d) && a.idx < b.idx); }

static int cmp_distidx(const void* a, const void* b) {
    DistIdx x = *(const DistIdx*)a, y = *(const DistIdx*)b;
    if (pair_less(x, y)) return -1;
    if (pair_less(y, x)) return 1;
    return 0;
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y);
}

/* ----------------------------------------------------------------- geometry */

/* proj/src/geometry.cpp:15-30 */
uint64_t orc_hilbert_index(uint32_t n, uint32_t x, uint32_t y) {
    uint64_t d = 0;
    for (uint32_t s = n / 2; s > 0; s /= 2) {
        uint32_t rx = (x & s) ? 1u : 0u;
        uint32_t ry = (y & s) ? 1u : 0u;
        d += (uint64_t)s * (uint64_t)s * ((3u * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            uint32_t t = x;
            x = y;
            y = t;
        }
    }
    return d;
}

/* min_gap, proj/src/geometry.cpp:57-65: smallest positive consecutive gap of
 * the sorted values, 0 if none */
static double min_gap(double* v, int64_t n) {
    qsort(v, (size_t)n, sizeof(double), cmp_double);
    double g = 0.0;
    for (int64_t i = 1; i < n; ++i) {
        double d = v[i] - v[i - 1];
        if (d > 0.0 && (g == 0.0 || d < g)) g = d;
    }
    return g;
}

/* proj/src/geometry.cpp:69-106.  std::stable_sort by key == sort of the
 * (key, index) pairs, which is what we do. */
int orc_sfc_order(const float* coords, int64_t n, int64_t* perm) {
    if (n < 1) return 2;
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    if (n == 1) return 0;
    double xmin = coords[0], xmax = xmin, ymin = coords[1], ymax = ymin;
    double* xs = (double*)malloc((size_t)n * sizeof(double));
    double* ys = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        xs[i] = coords[2 * i];
        ys[i] = coords[2 * i + 1];
        if (xs[i] < xmin) xmin = xs[i];
        if (xmax < xs[i]) xmax = xs[i];
        if (ys[i] < ymin) ymin = ys[i];
        if (ymax < ys[i]) ymax = ys[i];
    }
    double ex = xmax - xmin, ey = ymax - ymin;
    double extent = ex < ey ? ey : ex;
    if (extent <= 0.0) {
        free(xs);
        free(ys);
        return 0;
    }
    double gx = min_gap(xs, n), gy = min_gap(ys, n);
    double spacing = gx < gy ? gy : gx;
    if (spacing <= 0.0) spacing = extent;
    double arg = extent / spacing + 1.0;
    if (2.0 > arg) arg = 2.0; /* std::max(2.0, arg) */
    int b = (int)ceil(log2(arg));
    if (b < 1) b = 1;
    if (b > 16) b = 16;
    uint32_t side = 1u << b;
    double scale = (double)(side - 1) / extent;
    /* xs/ys were sorted by min_gap: re-read the coordinates */
    KeyIdx* ki = (KeyIdx*)malloc((size_t)n * sizeof(KeyIdx));
    for (int64_t i = 0; i < n; ++i) {
        uint32_t qx = (uint32_t)llround(((double)coords[2 * i] - xmin) * scale);
        uint32_t qy = (uint32_t)llround(((double)coords[2 * i + 1] - ymin) * scale);
        ki[i].key = orc_hilbert_index(side, qx, qy);
        ki[i].idx = i;
    }
    qsort(ki, (size_t)n, sizeof(KeyIdx), cmp_keyidx);
    for (int64_t i = 0; i < n; ++i) perm[i] = ki[i].idx;
    free(ki);
    free(xs);
    free(ys);
    return 0;
}

/* proj/src/geometry.cpp:108-131 */
int64_t orc_balanced_clusters(const float* coords, int64_t n, int64_t size, int32_t* cluster_of,
                              int64_t* members, int64_t* member_off) {
    if (size < 1) return -2;
    if (size > n) size = n;
    if (orc_sfc_order(coords, n, members) != 0) return -2;
    int64_t c = (n + size - 1) / size;
    int64_t base = n / c, rem = n % c, pos = 0;
    member_off[0] = 0;
    for (int64_t k = 0; k < c; ++k) {
        int64_t len = base + (k < rem ? 1 : 0);
        for (int64_t j = 0; j < len; ++j, ++pos) cluster_of[members[pos]] = (int32_t)k;
        member_off[k + 1] = pos;
    }
    return c;
}

/* proj/src/geometry.cpp:133-186 */
int orc_cluster_neighborhood(const float* coords, int64_t n, int64_t c, const int64_t* members,
                             const int64_t* member_off, int64_t groups, int64_t* nbr_cl,
                             int64_t* idx, uint8_t* valid, int64_t width) {
    if (groups < 1) return 2;
    if (groups > c) groups = c;
    double* cx = (double*)malloc((size_t)c * sizeof(double));
    double* cy = (double*)malloc((size_t)c * sizeof(double));
    int64_t max_size = 0;
    for (int64_t k = 0; k < c; ++k) {
        double sx = 0.0, sy = 0.0;
        for (int64_t p = member_off[k]; p < member_off[k + 1]; ++p) {
            sx += (double)coords[2 * members[p]];
            sy += (double)coords[2 * members[p] + 1];
        }
        int64_t len = member_off[k + 1] - member_off[k];
        double inv = 1.0 / (double)len;
        cx[k] = sx * inv;
        cy[k] = sy * inv;
        if (len > max_size) max_size = len;
    }
    int64_t m = groups * max_size;
    if (m > width) {
        free(cx);
        free(cy);
        return 2;
    }
    memset(idx, 0, (size_t)(n * width) * sizeof(int64_t));
    memset(valid, 0, (size_t)(n * width));
    DistIdx* best = (DistIdx*)malloc((size_t)groups * sizeof(DistIdx));
    for (int64_t k = 0; k < c; ++k) {
        /* the `groups` smallest (d^2, j) pairs, ascending (std::partial_sort) */
        int64_t nb = 0;
        for (int64_t j = 0; j < c; ++j) {
            double dx = cx[j] - cx[k];
            double dy = cy[j] - cy[k];
            DistIdx e = {dx * dx + dy * dy, j};
            if (nb < groups) {
                int64_t p = nb++;
                while (p > 0 && pair_less(e, best[p - 1])) {
                    best[p] = best[p - 1];
                    --p;
                }
                best[p] = e;
            } else if (pair_less(e, best[groups - 1])) {
                int64_t p = groups - 1;
                while (p > 0 && pair_less(e, best[p - 1])) {
                    best[p] = best[p - 1];
                    --p;
                }
                best[p] = e;
            }
        }
        /* own cluster first regardless of ties */
        int64_t* sel = nbr_cl + k * groups;
        int64_t ns = 0;
        sel[ns++] = k;
        for (int64_t g = 0; g < groups && ns < groups; ++g)
            if (best[g].idx != k) sel[ns++] = best[g].idx;
        for (int64_t p = member_off[k]; p < member_off[k + 1]; ++p) {
            int64_t t = members[p], s = 0;
            for (int64_t g = 0; g < groups; ++g)
                for (int64_t q = member_off[sel[g]]; q < member_off[sel[g] + 1]; ++q, ++s) {
                    idx[t * width + s] = members[q];
                    valid[t * width + s] = 1;
                }
        }
    }
    free(best);
    free(cx);
    free(cy);
    return 0;
}

/* proj/src/geometry.cpp:188-216 */
int orc_knn(const float* queries, int64_t nq, const float* keys, int64_t nk, int64_t k,
            int64_t* idx, uint8_t* valid) {
    if (nk < 1 || k < 1) return 2;
    int64_t kept = k < nk ? k : nk;
    memset(idx, 0, (size_t)(nq * k) * sizeof(int64_t));
    memset(valid, 0, (size_t)(nq * k));
    DistIdx* d = (DistIdx*)malloc((size_t)nk * sizeof(DistIdx));
    for (int64_t i = 0; i < nq; ++i) {
        double qx = queries[2 * i], qy = queries[2 * i + 1];
        for (int64_t j = 0; j < nk; ++j) {
            double dx = (double)keys[2 * j] - qx, dy = (double)keys[2 * j + 1] - qy;
            d[j].d = dx * dx + dy * dy;
            d[j].idx = j;
        }
        qsort(d, (size_t)nk, sizeof(DistIdx), cmp_distidx);
        for (int64_t s = 0; s < kept; ++s) {
            idx[i * k + s] = d[s].idx;
            valid[i * k + s] = 1;
        }
    }
    free(d);
    return 0;
}

/* ---------------------------------------------------------------- attention */

static double bias_eval_d(const double* w1, const double* b1, const double* w2, const double* b2,
                          int hidden, double patch, int h, double dx, double dy) {
    double ox = dx / patch, oy = dy / patch;
    double out = b2[h];
    for (int j = 0; j < hidden; ++j) {
        double pre = w1[h * 2 * hidden + j] * ox + w1[h * 2 * hidden + hidden + j] * oy +
                     b1[(int64_t)h * hidden + j];
        out += w2[(int64_t)h * hidden + j] * tanh(pre);
    }
    return out;
}

/* BiasNet::eval, proj/src/attention.cpp:33-42 */
double orc_bias_eval(const float* w1, const float* b1, const float* w2, const float* b2,
                     int hidden, double patch, int head, double dx, double dy) {
    double ox = dx / patch, oy = dy / patch;
    double out = b2[head];
    for (int j = 0; j < hidden; ++j) {
        double pre = (double)w1[head * 2 * hidden + j] * ox +
                     (double)w1[head * 2 * hidden + hidden + j] * oy +
                     (double)b1[(int64_t)head * hidden + j];
        out += (double)w2[(int64_t)head * hidden + j] * tanh(pre);
    }
    return out;
}

/* streaming_kernel<float>, proj/src/attention.cpp:119-185 (kTile = 16) */
int orc_attn_fwd_f32(int64_t n, int64_t m, int heads, int d, int hidden, double patch,
                     const float* q, const float* k, const float* v, const float* bk,
                     const float* bv, const float* coords, const int64_t* idx,
                     const uint8_t* valid, const float* w1, const float* b1, const float* w2,
                     const float* b2, const float* blank, float* out) {
    const int kTile = 16;
    int64_t slots = m + 1;
    int64_t hd = (int64_t)heads * d;
    double inv = 1.0 / sqrt((double)d);
    float invf = (float)inv;
    float* acc = (float*)malloc((size_t)d * sizeof(float));
    double s[16];
    for (int64_t i = 0; i < n; ++i) {
        double qx = coords[i * 2], qy = coords[i * 2 + 1];
        for (int h = 0; h < heads; ++h) {
            double run_max = NEG_INF;
            float l = 0.0f;
            for (int c = 0; c < d; ++c) acc[c] = 0.0f;
            for (int64_t t0 = 0; t0 < slots; t0 += kTile) {
                int64_t tn = slots - t0 < kTile ? slots - t0 : kTile;
                double tile_max = NEG_INF;
                for (int64_t j = 0; j < tn; ++j) {
                    int64_t slot = t0 + j;
                    if (slot < m && !valid[i * m + slot]) {
                        s[j] = NEG_INF;
                        continue;
                    }
                    float dot = 0.0f;
                    if (slot < m) {
                        int64_t key = idx[i * m + slot];
                        for (int c = 0; c < d; ++c)
                            dot += q[i * hd + h * d + c] * invf * k[key * hd + h * d + c];
                        double bias = orc_bias_eval(w1, b1, w2, b2, hidden, patch, h,
                                                    (double)coords[key * 2] - qx,
                                                    (double)coords[key * 2 + 1] - qy);
                        s[j] = (double)(float)((double)dot + bias);
                    } else {
                        for (int c = 0; c < d; ++c)
                            dot += q[i * hd + h * d + c] * invf * bk[(int64_t)h * d + c];
                        s[j] = (double)(float)((double)dot + (double)blank[h]);
                    }
                    tile_max = tile_max < s[j] ? s[j] : tile_max;
                }
                if (tile_max == NEG_INF) continue;
                double new_max = run_max < tile_max ? tile_max : run_max;
                float corr = run_max == NEG_INF ? 0.0f : expf((float)(run_max - new_max));
                l *= corr;
                for (int c = 0; c < d; ++c) acc[c] *= corr;
                for (int64_t j = 0; j < tn; ++j) {
                    if (s[j] == NEG_INF) continue;
                    int64_t slot = t0 + j;
                    float e = expf((float)(s[j] - new_max));
                    l += e;
                    if (slot < m) {
                        int64_t key = idx[i * m + slot];
                        for (int c = 0; c < d; ++c) acc[c] += e * v[key * hd + h * d + c];
                    } else {
                        for (int c = 0; c < d; ++c) acc[c] += e * bv[(int64_t)h * d + c];
                    }
                }
                run_max = new_max;
            }
            for (int c = 0; c < d; ++c) out[i * hd + h * d + c] = acc[c] / l;
        }
    }
    free(acc);
    return 0;
}

static inline void acc_store(double* a, int64_t i, double v, int prec) {
    a[i] = prec == 32 ? (double)(float)v : v;
}

/* nbhd_attn_backward, proj/src/attention.cpp:241-358 (score_row<double> at :67-88) */
int orc_attn_bwd(int64_t n, int64_t m, int heads, int d, int hidden, double patch, int prec,
                 const double* q, const double* k, const double* v, const double* bk,
                 const double* bv, const float* coords, const int64_t* idx,
                 const uint8_t* valid, const double* w1, const double* b1, const double* w2,
                 const double* b2, const double* blank, const double* dout, double* dq,
                 double* dk, double* dv, double* dbk, double* dbv, double* dw1, double* db1,
                 double* dw2, double* db2, double* dblank) {
    int64_t hd = (int64_t)heads * d;
    double inv = 1.0 / sqrt((double)d);
    memset(dq, 0, (size_t)(n * hd) * sizeof(double));
    memset(dk, 0, (size_t)(n * hd) * sizeof(double));
    memset(dv, 0, (size_t)(n * hd) * sizeof(double));
    memset(dbk, 0, (size_t)hd * sizeof(double));
    memset(dbv, 0, (size_t)hd * sizeof(double));
    memset(dw1, 0, (size_t)(heads * 2 * hidden) * sizeof(double));
    memset(db1, 0, (size_t)(heads * hidden) * sizeof(double));
    memset(dw2, 0, (size_t)(heads * hidden) * sizeof(double));
    memset(db2, 0, (size_t)heads * sizeof(double));
    memset(dblank, 0, (size_t)heads * sizeof(double));
    double* s = (double*)malloc((size_t)(m + 1) * sizeof(double));
    double* w = (double*)malloc((size_t)(m + 1) * sizeof(double));
    double* dwv = (double*)malloc((size_t)(m + 1) * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        double qx = coords[i * 2], qy = coords[i * 2 + 1];
        for (int h = 0; h < heads; ++h) {
            /* score_row<double> */
            for (int64_t j = 0; j <= m; ++j) s[j] = NEG_INF;
            for (int64_t j = 0; j < m; ++j) {
                if (!valid[i * m + j]) continue;
                int64_t key = idx[i * m + j];
                double acc = 0.0;
                for (int c = 0; c < d; ++c) acc += q[i * hd + h * d + c] * inv * k[key * hd + h * d + c];
                double bias = bias_eval_d(w1, b1, w2, b2, hidden, patch, h,
                                          (double)coords[key * 2] - qx,
                                          (double)coords[key * 2 + 1] - qy);
                s[j] = acc + bias;
            }
            {
                double acc = 0.0;
                for (int c = 0; c < d; ++c) acc += q[i * hd + h * d + c] * inv * bk[(int64_t)h * d + c];
                s[m] = acc + blank[h];
            }
            double mx = s[0];
            for (int64_t j = 1; j <= m; ++j)
                if (mx < s[j]) mx = s[j];
            double l = 0.0;
            for (int64_t j = 0; j <= m; ++j) {
                w[j] = 0.0;
                if (s[j] == NEG_INF) continue;
                w[j] = exp(s[j] - mx);
                l += w[j];
            }
            for (int64_t j = 0; j <= m; ++j) w[j] /= l;

            double wdot = 0.0;
            for (int64_t j = 0; j <= m; ++j) {
                dwv[j] = 0.0;
                if (w[j] == 0.0 && s[j] == NEG_INF) continue;
                double acc = 0.0;
                if (j < m) {
                    int64_t key = idx[i * m + j];
                    for (int c = 0; c < d; ++c) {
                        double go = dout[i * hd + h * d + c];
                        int64_t o = key * hd + h * d + c;
                        acc_store(dv, o, dv[o] + w[j] * go, prec);
                        acc += go * v[o];
                    }
                } else {
                    for (int c = 0; c < d; ++c) {
                        double go = dout[i * hd + h * d + c];
                        int64_t o = (int64_t)h * d + c;
                        acc_store(dbv, o, dbv[o] + w[j] * go, prec);
                        acc += go * bv[o];
                    }
                }
                dwv[j] = acc;
                wdot += w[j] * acc;
            }
            for (int64_t j = 0; j <= m; ++j) {
                if (s[j] == NEG_INF) continue;
                double ds = w[j] * (dwv[j] - wdot);
                if (ds == 0.0) continue;
                if (j < m) {
                    int64_t key = idx[i * m + j];
                    for (int c = 0; c < d; ++c) {
                        int64_t oi = i * hd + h * d + c, ok = key * hd + h * d + c;
                        acc_store(dq, oi, dq[oi] + ds * inv * k[ok], prec);
                        acc_store(dk, ok, dk[ok] + ds * inv * q[oi], prec);
                    }
                    double ox = ((double)coords[key * 2] - qx) / patch;
                    double oy = ((double)coords[key * 2 + 1] - qy) / patch;
                    for (int j2 = 0; j2 < hidden; ++j2) {
                        int64_t a = (int64_t)h * 2 * hidden + j2, b = (int64_t)h * hidden + j2;
                        double pre = w1[a] * ox + w1[a + hidden] * oy + b1[b];
                        double th = tanh(pre);
                        double w2v = w2[b];
                        double dpre = ds * w2v * (1.0 - th * th);
                        acc_store(dw2, b, dw2[b] + ds * th, prec);
                        acc_store(dw1, a, dw1[a] + dpre * ox, prec);
                        acc_store(dw1, a + hidden, dw1[a + hidden] + dpre * oy, prec);
                        acc_store(db1, b, db1[b] + dpre, prec);
                    }
                    acc_store(db2, h, db2[h] + ds, prec);
                } else {
                    for (int c = 0; c < d; ++c) {
                        int64_t oi = i * hd + h * d + c, ob = (int64_t)h * d + c;
                        acc_store(dq, oi, dq[oi] + ds * inv * bk[ob], prec);
                        acc_store(dbk, ob, dbk[ob] + ds * inv * q[oi], prec);
                    }
                    acc_store(dblank, h, dblank[h] + ds, prec);
                }
            }
        }
    }
    free(s);
    free(w);
    free(dwv);
    return 0;
}

/* ------------------------------------------------------------------ merging */

/* proj/src/merging.cpp:50-54 */
int64_t orc_retained_count(int64_t n, double d_s) {
    if (!(d_s > 0.0 && d_s <= 1.0)) return -2;
    int64_t k = (int64_t)floor(d_s * (double)n + 0.5);
    if (k > n) k = n;
    return k < 1 ? 1 : k;
}

typedef struct {
    double s;
    int64_t idx;
} ScoreIdx;

static int cmp_score_desc(const void* a, const void* b) {
    const ScoreIdx* x = (const ScoreIdx*)a;
    const ScoreIdx* y = (const ScoreIdx*)b;
    if (x->s != y->s) return x->s > y->s ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y);
}

/* proj/src/merging.cpp:56-69 */
int64_t orc_select_retained(const double* scores, int64_t n, double d_s, int64_t* out) {
    int64_t keep = orc_retained_count(n, d_s);
    if (keep < 0) return keep;
    ScoreIdx* o = (ScoreIdx*)malloc((size_t)n * sizeof(ScoreIdx));
    for (int64_t i = 0; i < n; ++i) {
        o[i].s = scores[i];
        o[i].idx = i;
    }
    qsort(o, (size_t)n, sizeof(ScoreIdx), cmp_score_desc);
    for (int64_t i = 0; i < keep; ++i) out[i] = o[i].idx;
    qsort(out, (size_t)keep, sizeof(int64_t), cmp_i64);
    free(o);
    return keep;
}

/* proj/src/merging.cpp:71-116 */
int orc_merge_plan(const float* coords, int64_t n, const int64_t* retained, int64_t r, int k_m,
                   int64_t* dropped, int64_t* target, int64_t* pool_idx, double* pool_dist,
                   int32_t* pool_cnt) {
    if (r < 1 || k_m < 1) return 2;
    uint8_t* is_ret = (uint8_t*)calloc((size_t)n, 1);
    for (int64_t i = 0; i < r; ++i) {
        if (retained[i] < 0 || retained[i] >= n) {
            free(is_ret);
            return 2;
        }
        is_ret[retained[i]] = 1;
    }
    int64_t* best_of = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    double* dist_of = (double*)malloc((size_t)n * sizeof(double));
    int64_t* cnt = (int64_t*)calloc((size_t)r, sizeof(int64_t));
    int64_t nd = 0;
    for (int64_t j = 0; j < n; ++j) {
        if (is_ret[j]) continue;
        double best = 0.0;
        int64_t best_r = -1;
        for (int64_t ri = 0; ri < r; ++ri) {
            double dx = (double)coords[2 * retained[ri]] - (double)coords[2 * j];
            double dy = (double)coords[2 * retained[ri] + 1] - (double)coords[2 * j + 1];
            double d2 = dx * dx + dy * dy;
            if (best_r < 0 || d2 < best) {
                best = d2;
                best_r = ri;
            }
        }
        dropped[nd] = j;
        target[nd] = retained[best_r];
        ++nd;
        best_of[j] = best_r;
        dist_of[j] = sqrt(best);
        cnt[best_r]++;
    }
    /* per-pool (dist, index) sort then truncation */
    int64_t* off = (int64_t*)malloc((size_t)(r + 1) * sizeof(int64_t));
    off[0] = 0;
    for (int64_t i = 0; i < r; ++i) off[i + 1] = off[i] + cnt[i];
    DistIdx* all = (DistIdx*)malloc((size_t)(nd > 0 ? nd : 1) * sizeof(DistIdx));
    int64_t* fill = (int64_t*)calloc((size_t)r, sizeof(int64_t));
    for (int64_t j = 0; j < n; ++j) {
        if (is_ret[j]) continue;
        int64_t ri = best_of[j];
        all[off[ri] + fill[ri]].d = dist_of[j];
        all[off[ri] + fill[ri]].idx = j;
        fill[ri]++;
    }
    for (int64_t ri = 0; ri < r; ++ri) {
        DistIdx* pl = all + off[ri];
        qsort(pl, (size_t)cnt[ri], sizeof(DistIdx), cmp_distidx);
        int64_t keep = cnt[ri] < k_m ? cnt[ri] : k_m;
        pool_cnt[ri] = (int32_t)keep;
        for (int64_t t = 0; t < k_m; ++t) {
            pool_idx[ri * k_m + t] = t < keep ? pl[t].idx : -1;
            pool_dist[ri * k_m + t] = t < keep ? pl[t].d : 0.0;
        }
    }
    free(is_ret);
    free(best_of);
    free(dist_of);
    free(cnt);
    free(off);
    free(all);
    free(fill);
    return 0;
}

/* pool_forward, proj/src/merging.cpp:121-149 */
int orc_merge_pool_fwd(int64_t n, int64_t dim, int64_t r, int k_m, int prec,
                       const int64_t* retained, const int64_t* pool_idx, const double* pool_dist,
                       const int32_t* pool_cnt, const double* feats, const double* scores,
                       double p, double* out) {
    (void)n;
    double w[64];
    if (k_m > 64) return 2;
    for (int64_t ri = 0; ri < r; ++ri) {
        int64_t rr = retained[ri], row = ri * 2 * dim;
        for (int64_t c = 0; c < dim; ++c) acc_store(out, row + c, feats[rr * dim + c], prec);
        int np = pool_cnt[ri];
        if (np == 0) {
            for (int64_t c = 0; c < dim; ++c) out[row + dim + c] = 0.0;
            continue;
        }
        const double* dist = pool_dist + ri * k_m;
        const int64_t* pool = pool_idx + ri * k_m;
        double mm = -p * dist[0];
        for (int t = 1; t < np; ++t) {
            double x = -p * dist[t];
            mm = mm < x ? x : mm;
        }
        double l = 0.0;
        for (int t = 0; t < np; ++t) {
            w[t] = exp(-p * dist[t] - mm);
            l += w[t];
        }
        for (int64_t c = 0; c < dim; ++c) {
            double acc = 0.0;
            for (int t = 0; t < np; ++t) acc += (w[t] / l) * scores[pool[t]] * feats[pool[t] * dim + c];
            acc_store(out, row + dim + c, acc, prec);
        }
    }
    return 0;
}

/* MergePoolOp::backward, proj/src/merging.cpp:169-219 */
int orc_merge_pool_bwd(int64_t n, int64_t dim, int64_t r, int k_m, int prec,
                       const int64_t* retained, const int64_t* pool_idx, const double* pool_dist,
                       const int32_t* pool_cnt, const double* feats, const double* scores,
                       double p, const double* dout, double* dfeats, double* dscores, double* dp) {
    (void)n;
    double w[64], dw[64];
    if (k_m > 64) return 2;
    for (int64_t ri = 0; ri < r; ++ri) {
        int64_t rr = retained[ri], row = ri * 2 * dim;
        if (dfeats)
            for (int64_t c = 0; c < dim; ++c)
                acc_store(dfeats, rr * dim + c, dfeats[rr * dim + c] + dout[row + c], prec);
        int np = pool_cnt[ri];
        if (np == 0) continue;
        const double* dist = pool_dist + ri * k_m;
        const int64_t* pool = pool_idx + ri * k_m;
        double mm = -p * dist[0];
        for (int t = 1; t < np; ++t) {
            double x = -p * dist[t];
            mm = mm < x ? x : mm;
        }
        double l = 0.0;
        for (int t = 0; t < np; ++t) {
            w[t] = exp(-p * dist[t] - mm);
            l += w[t];
        }
        for (int t = 0; t < np; ++t) w[t] /= l;
        for (int t = 0; t < np; ++t) {
            int64_t j = pool[t];
            double sj = scores[j];
            double dot = 0.0;
            for (int64_t c = 0; c < dim; ++c) {
                double go = dout[row + dim + c];
                dot += go * feats[j * dim + c];
                if (dfeats) acc_store(dfeats, j * dim + c, dfeats[j * dim + c] + go * w[t] * sj, prec);
            }
            if (dscores) acc_store(dscores, j, dscores[j] + w[t] * dot, prec);
            dw[t] = sj * dot;
        }
        double wdot = 0.0;
        for (int t = 0; t < np; ++t) wdot += w[t] * dw[t];
        if (dp) {
            double acc = 0.0;
            for (int t = 0; t < np; ++t) acc += w[t] * (dw[t] - wdot) * (-dist[t]);
            acc_store(dp, 0, dp[0] + acc, prec);
        }
    }
    return 0;
}

/* ---------------------------------------------------------------- interpolation
 * make_interp_op (proj/src/interpolation.cpp:192-251): per query, the valid
 * neighbours of its row; interp_softmax (:51-67) with `prec` rounding after
 * every step (cast_prec, :12-18; the distance d = sqrt(dx^2 + dy^2) + eps is
 * rounded once, :21-30), combine (:32-49); backward (:93-142) in binary64 with
 * the zero subgradient at an exact query/key coincidence. */
static inline double cprec(double v, int prec) { return prec == 32 ? (double)(float)v : v; }

int orc_interp_fwd(int64_t nq, int64_t dim, int64_t k, int prec, const double* queries, const float* key_coords,
                   const double* feats, const int64_t* idx, const uint8_t* valid, double p, double eps,
                   double* out) {
    double d[256], e[256];
    int64_t nb[256];
    if (k > 256) return 2;
    for (int64_t qi = 0; qi < nq; ++qi) {
        int64_t m = 0;
        for (int64_t t = 0; t < k; ++t)
            if (valid[qi * k + t]) nb[m++] = idx[qi * k + t];
        if (m == 0) return 2; /* ConfigError: no valid neighbors */
        const double qx = queries[2 * qi], qy = queries[2 * qi + 1];
        double mx = -INFINITY;
        for (int64_t i = 0; i < m; ++i) {
            double dx = qx - (double)key_coords[2 * nb[i]], dy = qy - (double)key_coords[2 * nb[i] + 1];
            d[i] = cprec(sqrt(dx * dx + dy * dy) + eps, prec);
            e[i] = cprec(-p * d[i], prec); /* logit */
            mx = e[i] > mx ? e[i] : mx;
        }
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            e[i] = cprec(exp(e[i] - mx), prec);
            s = cprec(s + e[i], prec);
        }
        for (int64_t i = 0; i < m; ++i) e[i] = cprec(e[i] / s, prec);
        for (int64_t c = 0; c < dim; ++c) {
            double acc = 0.0;
            for (int64_t i = 0; i < m; ++i) acc = cprec(acc + e[i] * feats[nb[i] * dim + c], prec);
            out[qi * dim + c] = acc;
        }
    }
    return 0;
}

int orc_interp_bwd(int64_t nq, int64_t dim, int64_t k, const double* queries, const float* key_coords,
                   const double* feats, const int64_t* idx, const uint8_t* valid, double p, double eps,
                   const double* dout, double* dfeats, double* dp, double* dq) {
    double r[256], d[256], w[256], dw[256];
    int64_t nb[256];
    if (k > 256) return 2;
    for (int64_t qi = 0; qi < nq; ++qi) {
        int64_t m = 0;
        for (int64_t t = 0; t < k; ++t)
            if (valid[qi * k + t]) nb[m++] = idx[qi * k + t];
        if (m == 0) return 2;
        const double qx = queries[2 * qi], qy = queries[2 * qi + 1];
        for (int64_t i = 0; i < m; ++i) {
            double dx = qx - (double)key_coords[2 * nb[i]], dy = qy - (double)key_coords[2 * nb[i] + 1];
            r[i] = sqrt(dx * dx + dy * dy);
            d[i] = r[i] + eps;
        }
        double mx = -p * d[0];
        for (int64_t i = 1; i < m; ++i) mx = mx > -p * d[i] ? mx : -p * d[i];
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            w[i] = exp(-p * d[i] - mx);
            s += w[i];
        }
        for (int64_t i = 0; i < m; ++i) w[i] /= s;
        const double* g = dout + qi * dim;
        for (int64_t i = 0; i < m; ++i) {
            double acc = 0.0;
            for (int64_t c = 0; c < dim; ++c) {
                dfeats[nb[i] * dim + c] += w[i] * g[c];
                acc += g[c] * feats[nb[i] * dim + c];
            }
            dw[i] = acc;
        }
        double wdot = 0.0, dpq = 0.0; /* per-query dp, then added (InterpOp::backward, :240) */
        for (int64_t i = 0; i < m; ++i) wdot += w[i] * dw[i];
        for (int64_t i = 0; i < m; ++i) {
            double dl = w[i] * (dw[i] - wdot);
            dpq += dl * (-d[i]);
            double dd = dl * (-p);
            if (r[i] > 0.0) {
                dq[2 * qi] += dd * (qx - (double)key_coords[2 * nb[i]]) / r[i];
                dq[2 * qi + 1] += dd * (qy - (double)key_coords[2 * nb[i] + 1]) / r[i];
            }
        }
        *dp += dpq;
    }
    return 0;
}

/* ---------------------------------------------------------------- AdamW
 * AdamW::lr_at / AdamW::step (proj/src/pipeline.cpp:643-680): linear warmup then
 * cosine; moments in binary64; decoupled decay for matrices only (rows > 1);
 * values stored at the tape precision (b32).  One step over n_params tensors
 * laid out back to back; m/v [P] carry the moments between calls. */
double orc_adamw_lr(double lr, int64_t warmup, int64_t total, int64_t step) {
    if (step < warmup) return lr * (double)(step + 1) / (double)warmup;
    int64_t span = total - warmup > 1 ? total - warmup : 1;
    double prog = (double)(step - warmup) / (double)span;
    prog = prog < 1.0 ? prog : 1.0;
    return lr * 0.5 * (1.0 + cos(3.14159265358979323846 * prog));
}

int orc_adamw_step(double lr, int64_t warmup, double wd, double beta1, double beta2, int64_t total, int64_t step,
                   int64_t n_params, const int64_t* rows, const int64_t* cols, const double* grad, double* value,
                   double* m, double* v) {
    const double a = orc_adamw_lr(lr, warmup, total, step), n = (double)(step + 1);
    const double bc1 = 1.0 - pow(beta1, n), bc2 = 1.0 - pow(beta2, n);
    int64_t o = 0;
    for (int64_t t = 0; t < n_params; ++t) {
        const int decay = rows[t] > 1;
        for (int64_t e = 0; e < rows[t] * cols[t]; ++e, ++o) {
            double g = grad[o];
            double mi = beta1 * m[o] + (1.0 - beta1) * g;
            double vi = beta2 * v[o] + (1.0 - beta2) * g * g;
            m[o] = mi;
            v[o] = vi;
            double upd = (mi / bc1) / (sqrt(vi / bc2) + 1e-8);
            double val = value[o];
            if (decay) val -= a * wd * val;
            value[o] = (double)(float)(val - a * upd);
        }
    }
    return 0;
}

