"""Parity at every point of the op sweep the bench claims (BASELINE configs[1]:
4k-64k visible tokens, D 64-256, K = 48), through the same device path the bench
times: device cluster index -> attention plan -> attention fwd/bwd, and
select_retained -> merge_plan -> pool fwd/bwd.

Above 16384 tokens/image two code paths switch (the index sort falls back to the
global radix sort, csrc/sort.cuh; select_retained to the score-key segmented
sort, csrc/merge.cu), so the 32761 / 65536 points pin code the smaller tests
never reach.  Indices are checked BIT-EXACT against the oracle restatement
(oracle/port, pinned to the reference by tests/golden); attention and pool
values within rel-L2 1e-2 (BASELINE north_star), on image 1 of a 2-image batch
(image offsets inside the batched kernels are exercised too).

References: proj/src/geometry.cpp:69-186, proj/src/merging.cpp:56-220,
proj/src/attention.cpp:119-358; proj/tests/acceptance.cpp:78-125.
"""
import numpy as np
import pytest

from oracle import port
from paper_2602_16249_b200.inputs import bf16_round
from tests.problems import attn_problem, lattice_coords, rel_l2

REL_TOL = 1e-2
GRIDS = {4096: 128, 8281: 182, 16384: 256, 32761: 362, 65536: 512}


def _dev(a, dt):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda").contiguous()


def _coords(n, batch=2, seed0=1000):
    c = lattice_coords(batch, GRIDS[n], seed0=seed0)
    assert c.shape[1] == n
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("n", sorted(GRIDS))
def test_sweep_index_select_plan_bit_exact(n):
    """Cluster index (perm, cluster_of, nbr_cl, reverse CSR), select_retained (with
    ties) and merge_plan (targets, pools, binary64 distances) at every sweep N."""
    import torch
    from paper_2602_16249_b200 import ops
    coords = _coords(n)
    B = coords.shape[0]
    index = ops.cluster_index(_dev(coords, torch.float32), 16, 3)
    rng = np.random.default_rng(n)
    scores = rng.uniform(0.1, 0.9, (B, n)).astype(np.float32)
    scores[:, ::5] = np.round(scores[:, ::5], 2)  # many exact ties
    ret = ops.select_retained(_dev(scores, torch.float32), 0.4)
    plan = ops.merge_plan(_dev(coords, torch.float32), ret, 8)
    torch.cuda.synchronize()
    perm, cof, nbr = (t.cpu().numpy() for t in (index.perm, index.cluster_of, index.nbr_cl))
    roff, rcl = index.rev_off.cpu().numpy(), index.rev_cl.cpu().numpy()
    ret = ret.cpu().numpy()
    tgt, pidx, pdist, pcnt = (t.cpu().numpy() for t in (plan.target, plan.pool_idx, plan.pool_dist,
                                                          plan.pool_cnt))
    for b in range(B):
        want = port.cluster_index(coords[b], 16, 3)
        np.testing.assert_array_equal(perm[b], want["members"], err_msg=f"perm image {b}")
        np.testing.assert_array_equal(cof[b], want["cluster_of"], err_msg=f"cluster_of image {b}")
        np.testing.assert_array_equal(nbr[b], want["nbr_cl"], err_msg=f"nbr_cl image {b}")
        C, G = want["nbr_cl"].shape
        cnt = np.bincount(want["nbr_cl"].ravel(), minlength=C)
        np.testing.assert_array_equal(roff[b], np.concatenate([[0], np.cumsum(cnt)]))
        # reverse lists: query clusters naming c', ascending
        order = np.argsort(want["nbr_cl"].ravel(), kind="stable")
        np.testing.assert_array_equal(rcl[b], (order // G).astype(np.int32))
        r = port.select_retained(scores[b].astype(np.float64), 0.4)
        np.testing.assert_array_equal(ret[b], r, err_msg=f"retained image {b}")
        pl = port.merge_plan(coords[b], r, 8)
        np.testing.assert_array_equal(tgt[b][pl["dropped"]], pl["target"], err_msg="target")
        np.testing.assert_array_equal(pcnt[b], pl["pool_cnt"], err_msg="pool_cnt")
        np.testing.assert_array_equal(pidx[b], pl["pool_idx"], err_msg="pool_idx")
        np.testing.assert_array_equal(pdist[b], pl["pool_dist"], err_msg="pool_dist")


ATTN_POINTS = [(4096, 64), (8281, 128), (16384, 256), (32761, 128), (32761, 256), (65536, 64),
               (65536, 256)]


def _attn_device(pb, index, geom, with_bwd=True):
    import torch
    from paper_2602_16249_b200 import ops
    bf = torch.bfloat16
    q, k, v, bk, bv = (_dev(pb[n], bf) for n in ("q", "k", "v", "bk", "bv"))
    c = _dev(pb["coords"], torch.float32)
    bias = ops.BiasNet.from_numpy(pb["bias"])
    plan = ops.attn_plan(geom, c, index, pb["heads"], pb["head_dim"], pb["hidden"])
    out, lse = ops.attn_fwd(geom, q, k, v, bk, bv, c, None, None, bias, pb["heads"], pb["head_dim"],
                            plan=plan)
    g = None
    if with_bwd:
        g = ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, pb["heads"], pb["head_dim"], out, lse,
                         _dev(pb["dout"], bf), plan=plan)
    torch.cuda.synchronize()
    return out, lse, g


def _check_image(pb, out, g, b, with_bwd=True):
    coords = pb["coords"]
    ci = port.cluster_index(coords[b], 16, 3)
    want = port.attn_fwd(pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"], coords[b], ci["idx"],
                         ci["valid"], pb["bias"], pb["heads"], pb["head_dim"])
    got = out[b].float().cpu().numpy()
    assert np.isfinite(got).all()
    err = {"out": rel_l2(got, want)}
    if with_bwd:
        wg = port.attn_bwd(pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"], coords[b], ci["idx"],
                           ci["valid"], pb["bias"], pb["heads"], pb["head_dim"], pb["dout"][b], prec=32)
        for n in ("dq", "dk", "dv"):
            err[n] = rel_l2(getattr(g, n)[b].float().cpu().numpy(), wg[n])
    return err


@pytest.mark.gpu
@pytest.mark.parametrize("n,dim", ATTN_POINTS, ids=[f"N{n}_D{d}" for n, d in ATTN_POINTS])
def test_sweep_attention_fwd_bwd(n, dim):
    """Attention fwd + dQ/dK/dV on the device-built index at the sweep's (N, D)
    points, head_dim 32 (h = D/32), BiasNet H = 8, image 1 of 2 vs the oracle."""
    import torch
    from paper_2602_16249_b200 import ops
    coords = _coords(n)
    rng = np.random.default_rng(n * 7 + dim)
    pb = attn_problem(coords, dim // 32, 32, 8, rng)
    geom = ops.geometry(2, n, 16, 3)
    index = ops.cluster_index(_dev(coords, torch.float32), 16, 3)
    out, _, g = _attn_device(pb, index, geom)
    err = _check_image(pb, out, g, 1)
    assert max(err.values()) <= REL_TOL, err


@pytest.mark.gpu
def test_bench_shape_attention_image31():
    """The bench's own shape: B = 32 images of a 256^2 grid (N = 16384), D = 128;
    the last image of the batch checked against the oracle (fwd + dQ/dK/dV)."""
    import torch
    from paper_2602_16249_b200 import ops
    coords = lattice_coords(32, 256, seed0=1000)
    rng = np.random.default_rng(2026)
    pb = attn_problem(coords, 4, 32, 8, rng)
    geom = ops.geometry(32, 16384, 16, 3)
    index = ops.cluster_index(_dev(coords, torch.float32), 16, 3)
    out, _, g = _attn_device(pb, index, geom)
    err = _check_image(pb, out, g, 31)
    assert max(err.values()) <= REL_TOL, err


@pytest.mark.gpu
@pytest.mark.parametrize("dup", ["pairs", "stacks"])
def test_attention_duplicate_coordinates(dup):
    """Duplicated coordinates (proj/tests/test_geometry.cpp:160-179 analogue): two
    tokens at one lattice cell make a key cell repeat inside a row, which takes the
    atomic fallback of the bias-table gradient.  Checks all ten gradients."""
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(99 if dup == "pairs" else 100)
    base = lattice_coords(2, 64, seed0=3)  # N = 1024
    c = base.copy()
    if dup == "pairs":
        c[:, 1::2] = c[:, 0::2]  # every odd token sits on its even neighbour
    else:
        c[:, :, :] = c[:, (np.arange(c.shape[1]) // 5) * 5, :]  # stacks of 5
    pb = attn_problem(np.ascontiguousarray(c), 4, 32, 8, rng)
    N = c.shape[1]
    geom = ops.geometry(2, N, 16, 3)
    index = ops.cluster_index(_dev(c, torch.float32), 16, 3)
    out, _, g = _attn_device(pb, index, geom)
    err = {}
    want_sum = None
    for b in range(2):
        ci = port.cluster_index(c[b], 16, 3)
        np.testing.assert_array_equal(index.perm[b].cpu().numpy(), ci["members"])
        wf = port.attn_fwd(pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"], c[b], ci["idx"],
                           ci["valid"], pb["bias"], 4, 32)
        err[f"out{b}"] = rel_l2(out[b].float().cpu().numpy(), wf)
        wg = port.attn_bwd(pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"], c[b], ci["idx"],
                           ci["valid"], pb["bias"], 4, 32, pb["dout"][b], prec=32)
        for n in ("dq", "dk", "dv"):
            err[f"{n}{b}"] = rel_l2(getattr(g, n)[b].float().cpu().numpy(), wg[n])
        shared = {n: wg[n] for n in ("dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank")}
        want_sum = shared if want_sum is None else {n: want_sum[n] + shared[n] for n in shared}
    for n, w in want_sum.items():
        err[n] = rel_l2(getattr(g, n).float().cpu().numpy().reshape(w.shape), w)
    assert max(err.values()) <= REL_TOL, err


@pytest.mark.gpu
@pytest.mark.parametrize("n,dim", [(32761, 256), (65536, 128)], ids=["N32761_D256", "N65536_D128"])
def test_sweep_pool_fwd_bwd(n, dim):
    """Merge pool fwd/bwd at the large sweep points (image 1 of 2)."""
    import torch
    from paper_2602_16249_b200 import ops
    coords = _coords(n)
    rng = np.random.default_rng(n + dim)
    scores = rng.uniform(0.1, 0.9, (2, n)).astype(np.float32)
    feats = bf16_round(rng.standard_normal((2, n, dim)).astype(np.float32))
    p = 1.0
    ret = ops.select_retained(_dev(scores, torch.float32), 0.4)
    plan = ops.merge_plan(_dev(coords, torch.float32), ret, 8)
    fd, sd, pd = _dev(feats, torch.bfloat16), _dev(scores, torch.float32), _dev([p], torch.float32)
    out = ops.merge_pool_fwd(fd, sd, pd, plan)
    R = ret.shape[1]
    dout = bf16_round(rng.standard_normal((2, R, 2 * dim)).astype(np.float32))
    df, ds, _ = ops.merge_pool_bwd(fd, sd, pd, plan, _dev(dout, torch.bfloat16))
    torch.cuda.synchronize()
    b = 1
    r = ret[b].cpu().numpy()
    pl = port.merge_plan(coords[b], r, 8)
    wo = port.merge_pool_fwd(pl, feats[b], scores[b], p)
    wdf, wds, _ = port.merge_pool_bwd(pl, feats[b], scores[b], p, dout[b])
    err = {"out": rel_l2(out[b].float().cpu().numpy(), wo), "dfeats": rel_l2(df[b].float().cpu().numpy(), wdf),
           "dscores": rel_l2(ds[b].cpu().numpy(), wds)}
    assert max(err.values()) <= REL_TOL, err
