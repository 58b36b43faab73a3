"""Generates the golden fixtures of tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libaffmae_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run here (the reference is not available on the GPU box):

    make -C oracle && python tests/golden/make_golden.py

Each fixture stores the inputs and the reference's outputs, so the CPU test suite
can pin the oracle restatement (oracle/oracle.c) without the reference present.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref  # noqa: E402


def rnd_points(rng, n, extent):
    return rng.uniform(0.0, extent, (n, 2)).astype(np.float32)


def main():
    out = {}
    rng = np.random.default_rng(20260217)
    # geometry: sfc order + clusters + neighbourhoods (proj/tests/test_geometry.cpp fixtures)
    cases = {"rand60_s8_g3": (rnd_points(rng, 60, 50.0), 8, 3),
             "rand100_s16_g3": (rnd_points(rng, 100, 100.0), 16, 3),
             "rand10_s8_g3": (rnd_points(rng, 10, 10.0), 8, 3),
             "dup5_s2_g3": (np.tile(np.array([[3.0, 7.0]], np.float32), (5, 1)), 2, 3),
             "grid64": (None, 16, 3)}
    mask = ref.perlin_mask(64, 0.75, 3)
    ys, xs = np.nonzero(mask == 0)
    cases["grid64"] = (np.stack([xs * 8 + 4, ys * 8 + 4], 1).astype(np.float32), 16, 3)
    out["perlin64_r075_s3"] = mask
    for name, (c, s, g) in cases.items():
        ci = ref.cluster_index(c, s, g)
        out[f"geo_{name}_coords"] = c
        out[f"geo_{name}_perm"] = ref.sfc_order(c)
        for k in ("cluster_of", "members", "member_off", "idx", "valid"):
            out[f"geo_{name}_{k}"] = ci[k]
        out[f"geo_{name}_shape"] = np.array([s, g])
    # knn with ties
    q = rnd_points(rng, 12, 20.0)
    keys = np.floor(rnd_points(rng, 40, 20.0))
    ki, kv = ref.knn(q, keys, 9)
    out.update(knn_q=q, knn_keys=keys, knn_idx=ki, knn_valid=kv)
    # attention (b32 streaming fwd, b32 and b64 backward), knn neighbourhoods with padding
    n, m, h, d, H = 40, 12, 2, 8, 4
    coords = rnd_points(rng, n, 64.0)
    idx, valid = ref.knn(coords, coords, m)
    valid[3, :] = 0
    valid[7, 5:] = 0
    f = lambda *s: rng.standard_normal(s)
    att = dict(q=f(n, h * d), k=f(n, h * d), v=f(n, h * d), bk=f(h, d), bv=f(h, d), dout=f(n, h * d),
               w1=0.7 * f(h, 2 * H), b1=0.3 * f(h, H), w2=0.7 * f(h, H), b2=0.3 * f(h, 1),
               blank=0.3 * f(h, 1))
    for k_, v_ in att.items():
        att[k_] = v_.astype(np.float32).astype(np.float64)  # b32-representable inputs
    bias = {k_: att[k_] for k_ in ("w1", "b1", "w2", "b2", "blank")}
    out.update({f"attn_{k_}": v_ for k_, v_ in att.items()})
    out.update(attn_coords=coords, attn_idx=idx, attn_valid=valid)
    out["attn_out_b32"] = ref.attn_fwd(att["q"], att["k"], att["v"], att["bk"], att["bv"], coords, idx,
                                       valid, bias, h, d, prec=32, mode=0)
    out["attn_out_naive_b64"] = ref.attn_fwd(att["q"], att["k"], att["v"], att["bk"], att["bv"], coords,
                                             idx, valid, bias, h, d, prec=64, mode=1)
    for prec in (32, 64):
        g = ref.attn_bwd(att["q"], att["k"], att["v"], att["bk"], att["bv"], coords, idx, valid, bias,
                         h, d, att["dout"], prec=prec)
        out.update({f"attn_grad{prec}_{k_}": v_ for k_, v_ in g.items()})
    # merging
    s6 = np.array([0.3, 0.9, 0.5, 0.9, 0.1, 0.5])
    out["sel_known_scores"] = s6
    out["sel_known_out"] = ref.select_retained(s6, 0.5)
    table = [(n_, ds) for ds in (0.25, 0.35, 0.4, 0.5, 1.0) for n_ in (1, 2, 7, 100, 4096)]
    out["retention_table"] = np.array([[n_, ds, ref.retained_count(n_, ds)] for n_, ds in table])
    for name, (npts, ext, ds, km) in {"m40": (40, 32.0, 0.35, 4), "m300": (300, 64.0, 0.4, 8),
                                       "m12": (12, 16.0, 0.4, 3)}.items():
        c = rnd_points(rng, npts, ext)
        sc = rng.uniform(0.1, 0.9, npts)
        r = ref.select_retained(sc, ds)
        pl = ref.merge_plan(c, r, km)
        feats = rng.standard_normal((npts, 5))
        po = ref.merge_pool_fwd(pl, feats, sc, 1.3)
        dd = rng.standard_normal(po.shape)
        df, dsc, dp = ref.merge_pool_bwd(pl, feats, sc, 1.3, dd)
        out.update({f"mrg_{name}_coords": c, f"mrg_{name}_scores": sc, f"mrg_{name}_retained": r,
                    f"mrg_{name}_feats": feats, f"mrg_{name}_dout": dd, f"mrg_{name}_pooled": po,
                    f"mrg_{name}_dfeats": df, f"mrg_{name}_dscores": dsc, f"mrg_{name}_dp": np.array([dp]),
                    f"mrg_{name}_dsk": np.array([ds, km])})
        for k_, v_ in pl.items():
            out[f"mrg_{name}_plan_{k_}"] = v_
    # make_interp_op (interpolation.cpp:192-251) on knn rows, b32 tape; own RNG so the
    # arrays above do not move when cases are added here
    irng = np.random.default_rng(2602)
    for name, (nk, nq, k, dim, p_) in {"i50": (50, 13, 6, 5, 1.5), "i200": (200, 40, 8, 7, 0.7)}.items():
        kc = rnd_points(irng, nk, 32.0)
        q = rnd_points(irng, nq, 32.0).astype(np.float64)
        q[0] = kc[3]  # exact query/key coincidence (zero subgradient)
        idx, valid = ref.knn(q.astype(np.float32), kc, k)
        valid[1, k // 2:] = 0  # a short row
        feats = irng.standard_normal((nk, dim)).astype(np.float32).astype(np.float64)
        dd = irng.standard_normal((nq, dim)).astype(np.float32).astype(np.float64)
        io = ref.interp_fwd(q, kc, feats, idx, valid, p_)
        df, dp, dq = ref.interp_bwd(q, kc, feats, idx, valid, p_, dd)
        out.update({f"itp_{name}_keys": kc, f"itp_{name}_queries": q, f"itp_{name}_idx": idx,
                    f"itp_{name}_valid": valid, f"itp_{name}_feats": feats, f"itp_{name}_dout": dd,
                    f"itp_{name}_p": np.array([p_]), f"itp_{name}_out": io, f"itp_{name}_dfeats": df,
                    f"itp_{name}_dp": np.array([dp]), f"itp_{name}_dq": dq})
    # AdamW (pipeline.cpp:639-680): matrices and vectors, warmup and cosine phases
    arng = np.random.default_rng(680)
    shapes = [(4, 6), (1, 6), (7, 3), (1, 1), (3, 1)]
    P = sum(a * b for a, b in shapes)
    vals = arng.standard_normal(P).astype(np.float32).astype(np.float64)
    grads = (arng.standard_normal((6, P)) * 0.1).astype(np.float32).astype(np.float64)
    out["adamw_shapes"] = np.array(shapes, np.int64)
    out["adamw_values"] = vals
    out["adamw_grads"] = grads
    out["adamw_out_w2_t6"] = ref.adamw(shapes, vals, grads, warmup=2, total=6)
    out["adamw_out_w100_t1000"] = ref.adamw(shapes, vals, grads, warmup=100, total=1000)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
