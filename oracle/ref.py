"""TEST INFRASTRUCTURE ONLY: ctypes view of oracle/_ref/libaffmae_ref.so.

That library is the UNMODIFIED reference C++ (``/root/reference/proj/src``)
compiled by ``oracle/Makefile`` plus our ``ref_shim.cpp``.  Only ``tests/``,
``__graft_entry__.smoke`` and ``bench.py``'s CPU legs may import this module;
the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libaffmae_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_retained_count.restype = C.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        if rc == 2:
            raise ValueError(msg)
        if rc == 3:
            raise ArithmeticError(msg)
        raise RuntimeError(msg)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def sfc_order(coords):
    coords = _f32(coords)
    n = coords.shape[0]
    perm = np.empty(n, np.int64)
    _check(lib().ref_sfc_order(_p(coords), C.c_int64(n), _p(perm)))
    return perm


def cluster_shape(n, size, groups):
    out = [C.c_int64() for _ in range(4)]
    _check(lib().ref_cluster_shape(C.c_int64(n), C.c_int64(size), C.c_int64(groups),
                                   *[C.byref(o) for o in out]))
    return tuple(o.value for o in out)  # (C, groups_eff, max_size, width)


def cluster_index(coords, size, groups):
    """balanced_clusters + cluster_neighborhood.

    Returns dict(cluster_of[n] i32, members[n] i64 (curve order), member_off[C+1],
    idx[n, M] i64, valid[n, M] u8, width M).
    """
    coords = _f32(coords)
    n = coords.shape[0]
    c, g, mx, width = cluster_shape(n, size, groups)
    cluster_of = np.empty(n, np.int32)
    members = np.empty(n, np.int64)
    off = np.empty(c + 1, np.int64)
    idx = np.empty((n, width), np.int64)
    valid = np.empty((n, width), np.uint8)
    _check(lib().ref_cluster_index(_p(coords), C.c_int64(n), C.c_int64(size), C.c_int64(groups),
                                   _p(cluster_of), _p(members), _p(off), _p(idx), _p(valid),
                                   C.c_int64(width)))
    return dict(cluster_of=cluster_of, members=members, member_off=off, idx=idx, valid=valid,
                width=width, n_clusters=c, groups=g, max_size=mx)


def knn(queries, keys, k):
    queries, keys = _f32(queries), _f32(keys)
    nq, nk = queries.shape[0], keys.shape[0]
    idx = np.empty((nq, k), np.int64)
    valid = np.empty((nq, k), np.uint8)
    _check(lib().ref_knn(_p(queries), C.c_int64(nq), _p(keys), C.c_int64(nk), C.c_int64(k),
                         _p(idx), _p(valid)))
    return idx, valid


def _attn_args(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, patch):
    q, k, v, bk, bv = (_f64(x) for x in (q, k, v, bk, bv))
    coords = _f32(coords)
    idx = _i64(idx)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    w1, b1, w2, b2, blank = (_f64(bias[x]) for x in ("w1", "b1", "w2", "b2", "blank"))
    n, m = idx.shape
    hidden = w1.shape[1] // 2
    keep = (q, k, v, bk, bv, coords, idx, valid, w1, b1, w2, b2, blank)
    args = [C.c_int64(n), C.c_int64(m), C.c_int(heads), C.c_int(head_dim), C.c_int(hidden),
            C.c_double(patch), _p(q), _p(k), _p(v), _p(bk), _p(bv), _p(coords), _p(idx),
            _p(valid), _p(w1), _p(b1), _p(w2), _p(b2), _p(blank)]
    return args, keep, n


def attn_fwd(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, patch=8.0, prec=32,
             mode=0):
    """nbhd_attn_streaming (mode 0), nbhd_attn_naive (1), streaming half_io (2)."""
    args, keep, n = _attn_args(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, patch)
    out = np.empty((n, heads * head_dim), np.float64)
    _check(lib().ref_attn_fwd(*args, C.c_int(prec), C.c_int(mode), _p(out)))
    return out


def attn_bwd(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, dout, patch=8.0,
             prec=32):
    args, keep, n = _attn_args(q, k, v, bk, bv, coords, idx, valid, bias, heads, head_dim, patch)
    dout = _f64(dout)
    hd = heads * head_dim
    hidden = keep[8].shape[1] // 2
    g = dict(dq=np.empty((n, hd)), dk=np.empty((n, hd)), dv=np.empty((n, hd)),
             dblank_k=np.empty((heads, head_dim)), dblank_v=np.empty((heads, head_dim)),
             dw1=np.empty((heads, 2 * hidden)), db1=np.empty((heads, hidden)),
             dw2=np.empty((heads, hidden)), db2=np.empty((heads, 1)), dblank=np.empty((heads, 1)))
    order = ("dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank")
    _check(lib().ref_attn_bwd(*args, C.c_int(prec), _p(dout), *[_p(g[o]) for o in order]))
    return g


def retained_count(n, d_s):
    r = lib().ref_retained_count(C.c_int64(n), C.c_double(d_s))
    if r < 0:
        raise ValueError(lib().ref_last_error().decode())
    return r


def select_retained(scores, d_s, prec=64):
    scores = _f64(scores).reshape(-1)
    n = scores.shape[0]
    out = np.empty(n, np.int64)
    cnt = C.c_int64()
    _check(lib().ref_select_retained(_p(scores), C.c_int64(n), C.c_double(d_s), C.c_int(prec),
                                     _p(out), C.byref(cnt)))
    return out[: cnt.value]


def merge_plan(coords, retained, k_m):
    coords = _f32(coords)
    retained = _i64(retained)
    n, r = coords.shape[0], retained.shape[0]
    dropped = np.empty(n - r, np.int64)
    target = np.empty(n - r, np.int64)
    pool_idx = np.empty((r, k_m), np.int64)
    pool_dist = np.empty((r, k_m), np.float64)
    pool_cnt = np.empty(r, np.int32)
    _check(lib().ref_merge_plan(_p(coords), C.c_int64(n), _p(retained), C.c_int64(r),
                                C.c_int(k_m), _p(dropped), _p(target), _p(pool_idx),
                                _p(pool_dist), _p(pool_cnt)))
    return dict(retained=retained, dropped=dropped, target=target, pool_idx=pool_idx,
                pool_dist=pool_dist, pool_cnt=pool_cnt)


def merge_pool_fwd(plan, feats, scores, p, prec=64):
    feats, scores = _f64(feats), _f64(scores).reshape(-1)
    n, dim = feats.shape
    r, k_m = plan["pool_idx"].shape
    out = np.empty((r, 2 * dim))
    _check(lib().ref_merge_pool_fwd(C.c_int64(n), C.c_int64(dim), C.c_int64(r), C.c_int(k_m),
                                    _p(_i64(plan["retained"])), _p(_i64(plan["pool_idx"])),
                                    _p(_f64(plan["pool_dist"])),
                                    _p(np.ascontiguousarray(plan["pool_cnt"], np.int32)),
                                    _p(feats), _p(scores), C.c_double(p), C.c_int(prec), _p(out)))
    return out


def importance_scores(feats, w1, b1, w2, b2, prec=32):
    """importance_scores (merging.cpp:31-48) of the compiled reference: feats [n, d],
    w1 [d, h], b1 [h], w2 [h], b2 scalar -> [n]."""
    feats = _f64(feats)
    n, d = feats.shape
    h = np.asarray(w1).shape[1]
    out = np.empty(n)
    _check(lib().ref_importance_scores(_p(feats), C.c_int64(n), C.c_int64(d), _p(_f64(w1)), _p(_f64(b1)),
                                       _p(_f64(w2)), C.c_double(float(b2)), C.c_int(h), C.c_int(prec), _p(out)))
    return out


def merge_tokens(coords, feats, scores, retained, k_m, p, proj_w, gamma, beta, prec=32):
    """merge_tokens (merging.cpp:242-273) of the compiled reference -> (coords [r, 2],
    feats [r, d])."""
    feats = _f64(feats)
    n, d = feats.shape
    r = len(retained)
    of, oc = np.empty((r, d)), np.empty((r, 2))
    _check(lib().ref_merge_tokens(_p(_f32(coords)), _p(feats), C.c_int64(n), C.c_int64(d),
                                  _p(_f64(scores).reshape(-1)), _p(_i64(retained)), C.c_int64(r), C.c_int(k_m),
                                  C.c_double(p), _p(_f64(proj_w)), _p(_f64(gamma)), _p(_f64(beta)), C.c_int(prec),
                                  _p(of), _p(oc)))
    return oc, of


def merge_pool_bwd(plan, feats, scores, p, dout, prec=64):
    feats, scores, dout = _f64(feats), _f64(scores).reshape(-1), _f64(dout)
    n, dim = feats.shape
    r, k_m = plan["pool_idx"].shape
    df = np.empty((n, dim))
    ds = np.empty(n)
    dp = C.c_double()
    keep = (_i64(plan["retained"]), _i64(plan["pool_idx"]), _f64(plan["pool_dist"]),
            np.ascontiguousarray(plan["pool_cnt"], np.int32))
    _check(lib().ref_merge_pool_bwd(C.c_int64(n), C.c_int64(dim), C.c_int64(r), C.c_int(k_m),
                                    *[_p(x) for x in keep], _p(feats), _p(scores), C.c_double(p),
                                    C.c_int(prec), _p(dout), _p(df), _p(ds), C.byref(dp)))
    return df, ds, dp.value


def interp_fwd(queries, key_coords, feats, idx, valid, p, eps=1e-6, prec=32):
    """make_interp_op forward (interpolation.cpp:192-222) of the compiled reference."""
    queries, feats = _f64(queries), _f64(feats)
    kc = _f32(key_coords)
    idx, valid = _i64(idx), np.ascontiguousarray(valid, np.uint8)
    nq, k = idx.shape
    nk, dim = feats.shape
    out = np.empty((nq, dim))
    _check(lib().ref_interp_fwd(C.c_int64(nq), C.c_int64(nk), C.c_int64(dim), C.c_int64(k), _p(queries),
                                _p(kc), _p(feats), _p(idx), _p(valid), C.c_double(p), C.c_double(eps),
                                C.c_int(prec), _p(out)))
    return out


def interp_bwd(queries, key_coords, feats, idx, valid, p, dout, eps=1e-6, prec=32):
    """make_interp_op backward (interpolation.cpp:224-251): dfeats, dp, dqueries."""
    queries, feats, dout = _f64(queries), _f64(feats), _f64(dout)
    kc = _f32(key_coords)
    idx, valid = _i64(idx), np.ascontiguousarray(valid, np.uint8)
    nq, k = idx.shape
    nk, dim = feats.shape
    df = np.empty((nk, dim))
    dq = np.empty((nq, 2))
    dp = C.c_double()
    _check(lib().ref_interp_bwd(C.c_int64(nq), C.c_int64(nk), C.c_int64(dim), C.c_int64(k), _p(queries),
                                _p(kc), _p(feats), _p(idx), _p(valid), C.c_double(p), C.c_double(eps),
                                C.c_int(prec), _p(dout), _p(df), C.byref(dp), _p(dq)))
    return df, dp.value, dq


def adamw(shapes, values, grads, lr=1e-3, warmup=100, wd=0.05, beta1=0.883, beta2=0.935, total=1000):
    """AdamW::step of the compiled reference, len(grads) steps; values/grads flat in tensor order."""
    rows = np.array([s[0] for s in shapes], np.int64)
    cols = np.array([s[1] for s in shapes], np.int64)
    vals = _f64(values).copy()
    g = _f64(grads)
    _check(lib().ref_adamw(C.c_double(lr), C.c_int64(warmup), C.c_double(wd), C.c_double(beta1),
                           C.c_double(beta2), C.c_int64(total), C.c_int64(len(shapes)), _p(rows), _p(cols),
                           C.c_int64(g.shape[0]), _p(g), _p(vals)))
    return vals


def synth_image(size, seed):
    out = np.empty(size * size)
    _check(lib().ref_synth_image(C.c_int64(size), C.c_uint64(seed), _p(out)))
    return out.reshape(size, size)


def write_aft(path, vals, prec=0):
    """write_aft (proj/src/tensor_io.cpp:60-66) of a tensor of precision `prec` (0 b32, 1 b16emu)."""
    vals = _f64(vals)
    dims = np.asarray(vals.shape, np.int64)
    _check(lib().ref_write_aft(path.encode(), _p(vals), _p(dims), C.c_int(vals.ndim), C.c_int(prec)))


def write_aft_u8(path, data):
    data = np.ascontiguousarray(data, np.uint8)
    dims = np.asarray(data.shape, np.int64)
    _check(lib().ref_write_aft_u8(path.encode(), _p(data), _p(dims), C.c_int(data.ndim)))


def read_aft(path, cap=1 << 24):
    """read_aft (proj/src/tensor_io.cpp:78-105): (flat float64 values, on-disk dtype code)."""
    out = np.empty(cap)
    n, dt = C.c_int64(), C.c_int()
    _check(lib().ref_read_aft(path.encode(), _p(out), C.c_int64(cap), C.byref(n), C.byref(dt)))
    return out[:n.value].copy(), dt.value


def load_checkpoint(directory, names, numels):
    """load_checkpoint (proj/src/pipeline.cpp:772-797) of the named parameters (flat
    float64 arrays); raises ValueError on the reference's ConfigError."""
    out = np.empty(int(sum(numels)))
    arr_names = (C.c_char_p * len(names))(*[n.encode() for n in names])
    nums = np.asarray(numels, np.int64)
    _check(lib().ref_load_checkpoint(str(directory).encode(), C.c_int(len(names)), arr_names, _p(nums), _p(out)))
    res, o = {}, 0
    for n, z in zip(names, numels):
        res[n] = out[o:o + z].copy()
        o += z
    return res


def perlin_mask(grid, ratio, seed):
    m = np.empty(grid * grid, np.uint8)
    _check(lib().ref_perlin_mask(C.c_int64(grid), C.c_double(ratio), C.c_uint64(seed), _p(m)))
    return m.reshape(grid, grid)


def hotpath_batch(images, threads, stages, coords, q, k, v, dout, scores, bk, bv, bias,
                  heads, head_dim, patch, cluster, groups, d_s, k_m, p):
    """Runs the reference hot path over `images` images on `threads` threads."""
    n = coords.shape[1]
    arrs = [_f32(coords)] + [_f64(x) for x in (q, k, v, dout, scores, bk, bv, bias["w1"],
                                               bias["b1"], bias["w2"], bias["b2"],
                                               bias["blank"])]
    hidden = arrs[8].shape[1] // 2
    cs = C.c_double()
    _check(lib().ref_hotpath_batch(C.c_int64(images), C.c_int(threads), C.c_int(stages),
                                   C.c_int64(n), C.c_int(heads), C.c_int(head_dim),
                                   C.c_int(hidden), C.c_double(patch), C.c_int64(cluster),
                                   C.c_int64(groups), C.c_double(d_s), C.c_int(k_m),
                                   *[_p(a) for a in arrs], C.c_double(p), C.byref(cs)))
    return cs.value


class RefModel:
    """The reference Model (proj/src/pipeline.cpp:255-746) through ref_shim.cpp, built from the
    same affmae_model_cfg struct the device model takes (paper_2602_16249_b200.model.ModelCfg)."""

    def __init__(self, cfg_struct, library=None):
        """library: a ctypes CDLL exporting the ref_model_* shim (default oracle/_ref; the
        drop-in test passes integration/libaffmae_model_b200.so -- the same reference Model
        with its hot-path calls on the B200 adapters)."""
        L = library or lib()
        if not hasattr(L, "ref_last_error") or L.ref_last_error.restype is not C.c_char_p:
            L.ref_last_error.restype = C.c_char_p
        self.L = L
        L.ref_model_create.restype = C.c_void_p
        L.ref_model_param_name.restype = C.c_char_p
        L.ref_model_param_numel.restype = C.c_int64
        for f in ("ref_model_destroy", "ref_model_param_count", "ref_model_param_name", "ref_model_param_numel",
                  "ref_model_get", "ref_model_set", "ref_model_fwd_bwd", "ref_model_train", "ref_model_make_mask"):
            getattr(L, f).argtypes = None
        self._cs = cfg_struct
        self.h = C.c_void_p(L.ref_model_create(C.byref(cfg_struct)))
        if not self.h.value:
            raise ValueError(L.ref_last_error().decode())
        n = L.ref_model_param_count(self.h)
        self.names = [L.ref_model_param_name(self.h, C.c_int(i)).decode() for i in range(n)]
        self.numel = [int(L.ref_model_param_numel(self.h, C.c_int(i))) for i in range(n)]

    def _check(self, rc):
        if rc != 0:
            msg = self.L.ref_last_error().decode()
            raise (ValueError if rc == 2 else ArithmeticError if rc == 3 else RuntimeError)(msg)

    def __del__(self):
        try:
            self.L.ref_model_destroy(self.h)
        except Exception:
            pass

    def _get(self, which):
        out = np.empty(int(sum(self.numel)))
        self._check(self.L.ref_model_get(self.h, C.c_int(which), _p(out)))
        res, o = {}, 0
        for n, z in zip(self.names, self.numel):
            res[n] = out[o:o + z].copy()
            o += z
        return res

    def params(self):
        return self._get(0)

    def grads(self):
        return self._get(1)

    def set_params(self, values):
        flat = np.concatenate([np.asarray(values[n], np.float64).ravel() for n in self.names])
        self._check(self.L.ref_model_set(self.h, _p(flat)))

    def fwd_bwd(self, image, masked, tokens_per_stage, dims):
        """-> ((total, main, aux), [coords of each stage], [stage features (pre-merge)]);
        the gradients are left in the model."""
        image = _f64(image)
        masked = np.ascontiguousarray(masked, np.uint8)
        loss = np.zeros(3)
        coords = np.zeros(int(sum(tokens_per_stage)) * 2, np.float32)
        feats = np.zeros(int(sum(n * d for n, d in zip(tokens_per_stage, dims))))
        self._check(self.L.ref_model_fwd_bwd(self.h, _p(image), C.c_int64(image.shape[0]), _p(masked), _p(loss),
                                       _p(coords), _p(feats)))
        co, fo, a, b = [], [], 0, 0
        for n, d in zip(tokens_per_stage, dims):
            co.append(coords[a:a + 2 * n].reshape(n, 2))
            fo.append(feats[b:b + n * d].reshape(n, d))
            a += 2 * n
            b += n * d
        return tuple(loss), co, fo

    def train(self, steps, images):
        images = _f64(images)
        losses = np.zeros(steps)
        self._check(self.L.ref_model_train(self.h, C.c_int64(steps), C.c_int64(images.shape[0]), _p(images),
                                     C.c_int64(images.shape[1]), _p(losses)))
        return losses

    def make_mask(self, seed):
        g = self._cs.image // self._cs.patch
        m = np.zeros(g * g, np.uint8)
        self._check(self.L.ref_model_make_mask(self.h, C.c_uint64(seed), _p(m)))
        return m.reshape(g, g)



_model_b200 = None


def model_b200_lib():
    """integration/libaffmae_model_b200.so: the reference's pipeline.cpp compiled unmodified
    with its hot-path calls redirected to the B200 adapters (integration/redirect_b200.hpp)."""
    global _model_b200
    if _model_b200 is None:
        path = os.path.join(os.path.dirname(_HERE), "integration", "libaffmae_model_b200.so")
        if not os.path.exists(path):
            raise RuntimeError(f"drop-in model library not built: {path} (make -C integration)")
        _model_b200 = C.CDLL(path)
        _model_b200.ref_last_error.restype = C.c_char_p
    return _model_b200


def model_train_threads(cfg_struct, threads, images_per_thread, image):
    image = _f64(image)
    cs = C.c_double()
    lib().ref_model_train_threads.argtypes = None
    _check(lib().ref_model_train_threads(C.byref(cfg_struct), C.c_int(threads), C.c_int64(images_per_thread),
                                         _p(image), C.c_int64(image.shape[0]), C.byref(cs)))
    return cs.value
