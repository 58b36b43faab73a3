"""TEST INFRASTRUCTURE ONLY: ctypes view of oracle/liboracle.so (the C restatement).

Same Python signatures as :mod:`oracle.ref` so tests can run either checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_hilbert_index.restype = C.c_uint64
        _lib.orc_hilbert_index.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        _lib.orc_balanced_clusters.restype = C.c_int64
        _lib.orc_retained_count.restype = C.c_int64
        _lib.orc_select_retained.restype = C.c_int64
        _lib.orc_bias_eval.restype = C.c_double
        _lib.orc_adamw_lr.restype = C.c_double
        _lib.orc_adamw_lr.argtypes = [C.c_double, C.c_int64, C.c_int64, C.c_int64]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc != 0:
        raise ValueError(f"oracle: configuration error (code {rc})")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def hilbert_index(n, x, y):
    return int(lib().orc_hilbert_index(n, x, y))


def sfc_order(coords):
    coords = _f32(coords)
    n = coords.shape[0]
    perm = np.empty(max(n, 1), np.int64)
    _check(lib().orc_sfc_order(_p(coords), C.c_int64(n), _p(perm)))
    return perm[:n]


def cluster_shape(n, size, groups):
    if size < 1 or groups < 1 or n < 1:
        raise ValueError("bad shape")
    s = min(size, n)
    c = (n + s - 1) // s
    g = min(groups, c)
    mx = n // c + (1 if n % c else 0)
    return c, g, mx, g * mx


def cluster_index(coords, size, groups):
    """balanced_clusters + cluster_neighborhood (same dict as oracle.ref.cluster_index,
    plus nbr_cl [C, groups_eff])."""
    coords = _f32(coords)
    n = coords.shape[0]
    c, g, mx, width = cluster_shape(n, size, groups)
    cluster_of = np.empty(n, np.int32)
    members = np.empty(n, np.int64)
    off = np.empty(c + 1, np.int64)
    cc = lib().orc_balanced_clusters(_p(coords), C.c_int64(n), C.c_int64(size), _p(cluster_of),
                                     _p(members), _p(off))
    if cc != c:
        raise ValueError("balanced_clusters failed")
    nbr_cl = np.empty((c, g), np.int64)
    idx = np.empty((n, width), np.int64)
    valid = np.empty((n, width), np.uint8)
    _check(lib().orc_cluster_neighborhood(_p(coords), C.c_int64(n), C.c_int64(c), _p(members),
                                          _p(off), C.c_int64(groups), _p(nbr_cl), _p(idx),
                                          _p(valid), C.c_int64(width)))
    return dict(cluster_of=cluster_of, members=members, member_off=off, idx=idx, valid=valid,
                width=width, n_clusters=c, groups=g, max_size=mx, nbr_cl=nbr_cl)


def knn(queries, keys, k):
    queries, keys = _f32(queries), _f32(keys)
    nq, nk = queries.shape[0], keys.shape[0]
    idx = np.empty((nq, k), np.int64)
    valid = np.empty((nq, k), np.uint8)
    _check(lib().orc_knn(_p(queries), C.c_int64(nq), _p(keys), C.c_int64(nk), C.c_int64(k),
                         _p(idx), _p(valid)))
    return idx, valid


def attn_fwd(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, patch=8.0):
    """streaming_kernel<float> on b32 tensors (inputs are cast to float32)."""
    q, k, v, bk, bv, coords = (_f32(x) for x in (q, k, v, bk, bv, coords))
    w1, b1, w2, b2, blank = (_f32(bias[x]) for x in ("w1", "b1", "w2", "b2", "blank"))
    idx = _i64(idx)
    valid = np.ascontiguousarray(valid, np.uint8)
    n, m = idx.shape
    hidden = w1.shape[1] // 2
    out = np.empty((n, heads * head_dim), np.float32)
    _check(lib().orc_attn_fwd_f32(C.c_int64(n), C.c_int64(m), C.c_int(heads), C.c_int(head_dim),
                                  C.c_int(hidden), C.c_double(patch), _p(q), _p(k), _p(v),
                                  _p(bk), _p(bv), _p(coords), _p(idx), _p(valid), _p(w1), _p(b1),
                                  _p(w2), _p(b2), _p(blank), _p(out)))
    return out


def attn_bwd(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, dout, patch=8.0,
             prec=32):
    """nbhd_attn_backward; prec=32 reproduces the b32 gradient tensors."""
    cast = _f32 if prec == 32 else _f64
    q, k, v, bk, bv, dout = (_f64(cast(x)) for x in (q, k, v, bk, bv, dout))
    w1, b1, w2, b2, blank = (_f64(cast(bias[x])) for x in ("w1", "b1", "w2", "b2", "blank"))
    coords = _f32(coords)
    idx = _i64(idx)
    valid = np.ascontiguousarray(valid, np.uint8)
    n, m = idx.shape
    hidden = w1.shape[1] // 2
    hd = heads * head_dim
    g = dict(dq=np.empty((n, hd)), dk=np.empty((n, hd)), dv=np.empty((n, hd)),
             dblank_k=np.empty((heads, head_dim)), dblank_v=np.empty((heads, head_dim)),
             dw1=np.empty((heads, 2 * hidden)), db1=np.empty((heads, hidden)),
             dw2=np.empty((heads, hidden)), db2=np.empty((heads, 1)), dblank=np.empty((heads, 1)))
    order = ("dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank")
    _check(lib().orc_attn_bwd(C.c_int64(n), C.c_int64(m), C.c_int(heads), C.c_int(head_dim),
                              C.c_int(hidden), C.c_double(patch), C.c_int(prec), _p(q), _p(k),
                              _p(v), _p(bk), _p(bv), _p(coords), _p(idx), _p(valid), _p(w1),
                              _p(b1), _p(w2), _p(b2), _p(blank), _p(dout),
                              *[_p(g[o]) for o in order]))
    return g


def retained_count(n, d_s):
    r = lib().orc_retained_count(C.c_int64(n), C.c_double(d_s))
    if r < 0:
        raise ValueError("retained_count: d_s must be in (0, 1]")
    return int(r)


def select_retained(scores, d_s):
    scores = _f64(scores).reshape(-1)
    n = scores.shape[0]
    out = np.empty(max(n, 1), np.int64)
    r = lib().orc_select_retained(_p(scores), C.c_int64(n), C.c_double(d_s), _p(out))
    if r < 0:
        raise ValueError("select_retained: d_s must be in (0, 1]")
    return out[:r]


def merge_plan(coords, retained, k_m):
    coords = _f32(coords)
    retained = _i64(retained)
    n, r = coords.shape[0], retained.shape[0]
    dropped = np.empty(max(n - r, 1), np.int64)
    target = np.empty(max(n - r, 1), np.int64)
    pool_idx = np.empty((r, k_m), np.int64)
    pool_dist = np.empty((r, k_m), np.float64)
    pool_cnt = np.empty(r, np.int32)
    _check(lib().orc_merge_plan(_p(coords), C.c_int64(n), _p(retained), C.c_int64(r),
                                C.c_int(k_m), _p(dropped), _p(target), _p(pool_idx),
                                _p(pool_dist), _p(pool_cnt)))
    return dict(retained=retained, dropped=dropped[: n - r], target=target[: n - r],
                pool_idx=pool_idx, pool_dist=pool_dist, pool_cnt=pool_cnt)


def _plan_args(plan):
    return (_i64(plan["retained"]), _i64(plan["pool_idx"]), _f64(plan["pool_dist"]),
            np.ascontiguousarray(plan["pool_cnt"], np.int32))


def merge_pool_fwd(plan, feats, scores, p, prec=64):
    feats, scores = _f64(feats), _f64(scores).reshape(-1)
    n, dim = feats.shape
    r, k_m = plan["pool_idx"].shape
    out = np.empty((r, 2 * dim))
    pa = _plan_args(plan)
    _check(lib().orc_merge_pool_fwd(C.c_int64(n), C.c_int64(dim), C.c_int64(r), C.c_int(k_m),
                                    C.c_int(prec), *[_p(x) for x in pa], _p(feats), _p(scores),
                                    C.c_double(p), _p(out)))
    return out


def merge_pool_bwd(plan, feats, scores, p, dout, prec=64):
    feats, scores, dout = _f64(feats), _f64(scores).reshape(-1), _f64(dout)
    n, dim = feats.shape
    r, k_m = plan["pool_idx"].shape
    df = np.zeros((n, dim))
    ds = np.zeros(n)
    dp = np.zeros(1)
    pa = _plan_args(plan)
    _check(lib().orc_merge_pool_bwd(C.c_int64(n), C.c_int64(dim), C.c_int64(r), C.c_int(k_m),
                                    C.c_int(prec), *[_p(x) for x in pa], _p(feats), _p(scores),
                                    C.c_double(p), _p(dout), _p(df), _p(ds), _p(dp)))
    return df, ds, float(dp[0])


def interp_fwd(queries, key_coords, feats, idx, valid, p, eps=1e-6, prec=32):
    """make_interp_op forward (interpolation.cpp:192-222) restated in oracle.c.  The
    temperature is a tape tensor, so at b32 it is the float-rounded p."""
    p = float(np.float32(p)) if prec == 32 else float(p)
    queries, feats = _f64(queries), _f64(feats)
    kc = _f32(key_coords)
    idx, valid = _i64(idx), np.ascontiguousarray(valid, np.uint8)
    nq, k = idx.shape
    dim = feats.shape[1]
    out = np.empty((nq, dim))
    _check(lib().orc_interp_fwd(C.c_int64(nq), C.c_int64(dim), C.c_int64(k), C.c_int(prec), _p(queries), _p(kc),
                                _p(feats), _p(idx), _p(valid), C.c_double(p), C.c_double(eps), _p(out)))
    return out


def interp_bwd(queries, key_coords, feats, idx, valid, p, dout, eps=1e-6, prec=32):
    """make_interp_op backward (interpolation.cpp:224-251, binary64 math on the tape's
    values): dfeats, dp, dqueries."""
    p = float(np.float32(p)) if prec == 32 else float(p)
    queries, feats, dout = _f64(queries), _f64(feats), _f64(dout)
    kc = _f32(key_coords)
    idx, valid = _i64(idx), np.ascontiguousarray(valid, np.uint8)
    nq, k = idx.shape
    dim = feats.shape[1]
    df = np.zeros(feats.shape)
    dq = np.zeros((nq, 2))
    dp = np.zeros(1)
    _check(lib().orc_interp_bwd(C.c_int64(nq), C.c_int64(dim), C.c_int64(k), _p(queries), _p(kc), _p(feats),
                                _p(idx), _p(valid), C.c_double(p), C.c_double(eps), _p(dout), _p(df), _p(dp),
                                _p(dq)))
    return df, float(dp[0]), dq



def adamw(shapes, values, grads, lr=1e-3, warmup=100, wd=0.05, beta1=0.883, beta2=0.935, total=1000):
    """AdamW::step (pipeline.cpp:650-680) restated in oracle.c, len(grads) steps from zero moments;
    returns the values and the binary64 moments."""
    rows = np.array([s[0] for s in shapes], np.int64)
    cols = np.array([s[1] for s in shapes], np.int64)
    vals = _f64(values).copy()
    m = np.zeros_like(vals)
    v = np.zeros_like(vals)
    for st, g in enumerate(_f64(grads)):
        g = np.ascontiguousarray(g.astype(np.float32).astype(np.float64))  # grads live at b32 on the tape
        _check(lib().orc_adamw_step(C.c_double(lr), C.c_int64(warmup), C.c_double(wd), C.c_double(beta1),
                                    C.c_double(beta2), C.c_int64(total), C.c_int64(st), C.c_int64(len(shapes)),
                                    _p(rows), _p(cols), _p(g), _p(vals), _p(m), _p(v)))
    return vals, m, v
