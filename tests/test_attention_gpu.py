"""Cluster attention parity: CUDA (through the C ABI) vs the oracle restatement of
nbhd_attn_streaming / nbhd_attn_backward (proj/src/attention.cpp:119-358).

Tolerance (BASELINE north_star): bf16 inputs, fp32 accumulate;
outputs and gradients within rel-L2 <= 1e-2 of the b32 oracle run on the same
bf16-rounded inputs.  Max-abs error is also bounded loosely (0.05) to catch
isolated bad rows that an L2 norm would hide.
"""
import zlib

import numpy as np
import pytest

from oracle import port
from tests.problems import attn_problem, lattice_coords, random_coords, rel_l2

REL_TOL = 1e-2
ABS_TOL = 5e-2


def _torch():
    import torch
    return torch


def _host_index(coords, cluster, groups):
    """Cluster index of each image from the oracle (independent of the GPU index
    builder): perm, cluster_of, nbr_cl and the reverse-neighbour CSR."""
    perms, cofs, nbrs, roffs, rcls = [], [], [], [], []
    for b in range(coords.shape[0]):
        ci = port.cluster_index(coords[b], cluster, groups)
        nb = ci["nbr_cl"]
        C, G = nb.shape
        rev = [[] for _ in range(C)]
        for c in range(C):
            for g in range(G):
                rev[nb[c, g]].append(c)
        roffs.append(np.cumsum([0] + [len(r) for r in rev]))
        rcls.append(np.array([c for r in rev for c in r]))
        perms.append(ci["members"])
        cofs.append(ci["cluster_of"])
        nbrs.append(nb)
    st = lambda xs: np.stack(xs).astype(np.int32)
    return st(perms), st(cofs), st(nbrs), st(roffs), st(rcls)


def _dev(a, dt):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda").contiguous()


def _run_fwd(pb, cluster, groups):
    torch = _torch()
    from paper_2602_16249_b200 import ops
    coords = pb["coords"]
    B, N, _ = coords.shape
    geom = ops.geometry(B, N, cluster, groups)
    perm, _, nbr, _, _ = _host_index(coords, cluster, groups)
    dev = _dev
    bias = ops.BiasNet.from_numpy(pb["bias"])
    out, lse = ops.attn_fwd(geom, dev(pb["q"], torch.bfloat16), dev(pb["k"], torch.bfloat16),
                            dev(pb["v"], torch.bfloat16), dev(pb["bk"], torch.bfloat16),
                            dev(pb["bv"], torch.bfloat16), dev(coords, torch.float32),
                            dev(perm, torch.int32), dev(nbr, torch.int32), bias, pb["heads"],
                            pb["head_dim"])
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), lse.cpu().numpy()


def _oracle_fwd(pb, cluster, groups):
    outs = []
    for b in range(pb["coords"].shape[0]):
        ci = port.cluster_index(pb["coords"][b], cluster, groups)
        outs.append(port.attn_fwd(pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"],
                                  pb["coords"][b], ci["idx"], ci["valid"], pb["bias"],
                                  pb["heads"], pb["head_dim"]))
    return np.stack(outs)


CASES = [
    # (name, coords-maker, heads, head_dim, hidden, cluster, groups)
    ("lattice128_h4d32", lambda rng: lattice_coords(2, 128), 4, 32, 8, 16, 3),
    ("lattice64_h2d32", lambda rng: lattice_coords(3, 64, seed0=7), 2, 32, 8, 16, 3),
    ("random_h1d64", lambda rng: random_coords(2, 300, 64.0, rng), 1, 64, 4, 16, 3),
    ("random_h8d16", lambda rng: random_coords(2, 250, 100.0, rng), 8, 16, 8, 8, 3),
    ("ragged_h4d32", lambda rng: random_coords(2, 1001, 200.0, rng), 4, 32, 8, 16, 3),
    ("tiny_fewer_clusters", lambda rng: random_coords(1, 10, 10.0, rng), 2, 16, 4, 8, 3),
    ("toy_stage1", lambda rng: random_coords(2, 77, 64.0, rng), 4, 16, 8, 8, 3),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_attn_fwd_matches_oracle(case):
    name, mk, heads, hd, hidden, cluster, groups = case
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    pb = attn_problem(mk(rng), heads, hd, hidden, rng)
    got, lse = _run_fwd(pb, cluster, groups)
    want = _oracle_fwd(pb, cluster, groups)
    assert np.isfinite(got).all() and np.isfinite(lse).all()
    err = rel_l2(got, want)
    assert err <= REL_TOL, f"rel-L2 {err:.3e}"
    assert np.abs(got - want).max() <= ABS_TOL


@pytest.mark.gpu
def test_attn_fwd_single_cluster_blank_only_fallback():
    """A neighbourhood that holds only the query itself plus the blank: with a
    huge negative bias on real keys the output falls back to blank_v
    (proj/tests/test_attention.cpp:146-156 analogue)."""
    rng = np.random.default_rng(5)
    pb = attn_problem(random_coords(1, 16, 32.0, rng), 2, 32, 4, rng)
    pb["bias"]["b2"][:] = -1e4  # every real key slot -> exp(-huge) = 0
    got, _ = _run_fwd(pb, 16, 3)
    want = np.broadcast_to(pb["bv"].reshape(1, 1, -1), got.shape)
    assert np.abs(got - want).max() <= 1e-2


def _run_fwd_bwd(pb, cluster, groups):
    torch = _torch()
    from paper_2602_16249_b200 import ops
    coords = pb["coords"]
    B, N, _ = coords.shape
    geom = ops.geometry(B, N, cluster, groups)
    perm, cof, nbr, roff, rcl = (_dev(a, torch.int32) for a in _host_index(coords, cluster, groups))
    index = ops.ClusterIndex(geom, perm, cof, nbr, roff, rcl)
    bf = torch.bfloat16
    q, k, v, bk, bv = (_dev(pb[n], bf) for n in ("q", "k", "v", "bk", "bv"))
    c = _dev(coords, torch.float32)
    bias = ops.BiasNet.from_numpy(pb["bias"])
    out, lse = ops.attn_fwd(geom, q, k, v, bk, bv, c, perm, nbr, bias, pb["heads"], pb["head_dim"])
    g = ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, pb["heads"], pb["head_dim"], out, lse,
                     _dev(pb["dout"], bf))
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    return {n: f(getattr(g, n)) for n in ("dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1",
                                          "dw2", "db2", "dblank")}


def _oracle_bwd(pb, cluster, groups):
    acc = None
    per_img = {"dq": [], "dk": [], "dv": []}
    for b in range(pb["coords"].shape[0]):
        ci = port.cluster_index(pb["coords"][b], cluster, groups)
        g = port.attn_bwd(pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"],
                          pb["coords"][b], ci["idx"], ci["valid"], pb["bias"], pb["heads"],
                          pb["head_dim"], pb["dout"][b], prec=32)
        for n in per_img:
            per_img[n].append(g[n])
        if acc is None:
            acc = {n: g[n].copy() for n in g if n not in per_img}
        else:
            for n in acc:
                acc[n] += g[n]
    acc.update({n: np.stack(v) for n, v in per_img.items()})
    return acc


BWD_CASES = [CASES[0], CASES[1], CASES[2], CASES[3], CASES[4], CASES[6]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", BWD_CASES, ids=[c[0] for c in BWD_CASES])
def test_attn_bwd_matches_oracle(case):
    name, mk, heads, hd, hidden, cluster, groups = case
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    pb = attn_problem(mk(rng), heads, hd, hidden, rng)
    got = _run_fwd_bwd(pb, cluster, groups)
    want = _oracle_bwd(pb, cluster, groups)
    report = {}
    for n in want:
        g, w = got[n].reshape(want[n].shape), want[n]
        assert np.isfinite(g).all(), n
        report[n] = rel_l2(g, w)
    bad = {n: e for n, e in report.items() if e > REL_TOL}
    assert not bad, f"rel-L2 over {REL_TOL}: {bad} (all: {report})"


@pytest.mark.gpu
@pytest.mark.parametrize("case", [CASES[0], CASES[3]], ids=[CASES[0][0], CASES[3][0]])
def test_attn_planned_equals_oneshot(case):
    """The plan API (built once per cluster index, like the reference AttnOp freezing its
    geometry) gives bit-identical outputs and gradients to the one-shot calls."""
    torch = _torch()
    from paper_2602_16249_b200 import ops
    name, mk, heads, hd, hidden, cluster, groups = case
    rng = np.random.default_rng(zlib.crc32(name.encode()) + 1)
    pb = attn_problem(mk(rng), heads, hd, hidden, rng)
    coords = pb["coords"]
    B, N, _ = coords.shape
    geom = ops.geometry(B, N, cluster, groups)
    perm, cof, nbr, roff, rcl = (_dev(a, torch.int32) for a in _host_index(coords, cluster, groups))
    index = ops.ClusterIndex(geom, perm, cof, nbr, roff, rcl)
    bf = torch.bfloat16
    q, k, v, bk, bv = (_dev(pb[n], bf) for n in ("q", "k", "v", "bk", "bv"))
    c = _dev(coords, torch.float32)
    do = _dev(pb["dout"], bf)
    bias = ops.BiasNet.from_numpy(pb["bias"])
    o1, l1 = ops.attn_fwd(geom, q, k, v, bk, bv, c, perm, nbr, bias, heads, hd)
    g1 = ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, heads, hd, o1, l1, do)
    plan = ops.attn_plan(geom, c, index, heads, hd, hidden)
    o2, l2 = ops.attn_fwd(geom, q, k, v, bk, bv, c, None, None, bias, heads, hd, plan=plan)
    g2 = ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, heads, hd, o2, l2, do, plan=plan)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for n in ("dq", "dk", "dv", "dblank_k", "dblank_v", "dblank"):
        assert torch.equal(getattr(g1, n), getattr(g2, n)), n
    # BiasNet parameter gradients: far same-phase pairs (beyond the shared window)
    # accumulate through global atomics, so only the summation order may differ
    for n in ("dw1", "db1", "dw2", "db2"):
        assert torch.allclose(getattr(g1, n), getattr(g2, n), rtol=1e-5, atol=1e-5), n


@pytest.mark.gpu
def test_attn_plan_mismatch_raises():
    torch = _torch()
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(3)
    pb = attn_problem(lattice_coords(1, 32), 2, 32, 8, rng)
    coords = pb["coords"]
    B, N, _ = coords.shape
    geom = ops.geometry(B, N, 16, 3)
    perm, cof, nbr, roff, rcl = (_dev(a, torch.int32) for a in _host_index(coords, 16, 3))
    index = ops.ClusterIndex(geom, perm, cof, nbr, roff, rcl)
    c = _dev(coords, torch.float32)
    fwd_only = ops.attn_plan(geom, c, index, 2, 32, 8, with_reverse=False)
    bf = torch.bfloat16
    q = _dev(pb["q"], bf)
    bias = ops.BiasNet.from_numpy(pb["bias"])
    bk = _dev(pb["bk"], bf)
    o, l = ops.attn_fwd(geom, q, q, q, bk, bk, c, None, None, bias, 2, 32, plan=fwd_only)
    with pytest.raises(ValueError):  # backward needs the reverse CSR
        ops.attn_bwd(geom, q, q, q, bk, bk, c, index, bias, 2, 32, o, l, q, plan=fwd_only)
    other = ops.geometry(B, N, 8, 3)
    with pytest.raises(ValueError):  # plan built for another geometry
        ops.attn_fwd(other, q, q, q, bk, bk, c, None, None, bias, 2, 32, plan=fwd_only)
