"""Merge parity: select_retained / merge_plan bit-exact, merge pool fwd/bwd within
bf16 tolerance, against the oracle restatement of proj/src/merging.cpp:50-220
(known answers from proj/tests/test_merging.cpp)."""
import zlib

import numpy as np
import pytest

from oracle import port
from paper_2602_16249_b200.inputs import bf16_round
from tests.problems import lattice_coords, random_coords, rel_l2


def _dev(a, dt):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


@pytest.mark.gpu
def test_select_retained_known_answer():
    """{0.3,0.9,0.5,0.9,0.1,0.5} @ 0.5 -> {1,2,3} (proj/tests/test_merging.cpp:61-71)."""
    import torch
    from paper_2602_16249_b200 import ops
    s = _dev([[0.3, 0.9, 0.5, 0.9, 0.1, 0.5]], torch.float32)
    assert ops.select_retained(s, 0.5).cpu().numpy().tolist() == [[1, 2, 3]]


@pytest.mark.gpu
@pytest.mark.parametrize("n,d_s", [(1, 0.25), (7, 0.35), (100, 0.4), (4096, 0.4), (16384, 0.4),
                                   (1000, 1.0), (333, 0.5)])
def test_select_retained_bit_exact(n, d_s):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(n)
    s = rng.uniform(0.1, 0.9, (3, n)).astype(np.float32)
    s[:, ::7] = np.round(s[:, ::7], 1)  # ties
    got = ops.select_retained(_dev(s, torch.float32), d_s).cpu().numpy()
    for b in range(3):
        np.testing.assert_array_equal(got[b], port.select_retained(s[b].astype(np.float64), d_s))


PLAN_CASES = [
    ("lattice256", lambda rng: lattice_coords(3, 256), 0.4, 8),
    ("lattice128", lambda rng: lattice_coords(2, 128, seed0=5), 0.4, 8),
    ("random", lambda rng: random_coords(2, 2000, 100.0, rng), 0.4, 8),
    ("random_km3", lambda rng: random_coords(2, 40, 32.0, rng), 0.35, 3),
    ("clumped", lambda rng: np.floor(random_coords(2, 600, 12.0, rng)).astype(np.float32), 0.3, 5),
    ("tiny", lambda rng: random_coords(1, 3, 4.0, rng), 0.4, 8),
]


def _plan_problem(name, mk, d_s):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    coords = np.ascontiguousarray(mk(rng), dtype=np.float32)
    B, N, _ = coords.shape
    scores = rng.uniform(0.1, 0.9, (B, N)).astype(np.float32)
    return rng, coords, scores


@pytest.mark.gpu
@pytest.mark.parametrize("case", PLAN_CASES, ids=[c[0] for c in PLAN_CASES])
def test_merge_plan_bit_exact(case):
    import torch
    from paper_2602_16249_b200 import ops
    name, mk, d_s, k_m = case
    rng, coords, scores = _plan_problem(name, mk, d_s)
    B, N, _ = coords.shape
    ret = ops.select_retained(_dev(scores, torch.float32), d_s)
    plan = ops.merge_plan(_dev(coords, torch.float32), ret, k_m)
    torch.cuda.synchronize()
    tgt = plan.target.cpu().numpy()
    pidx, pdist, pcnt = (t.cpu().numpy() for t in (plan.pool_idx, plan.pool_dist, plan.pool_cnt))
    row_of = plan.row_of.cpu().numpy()
    for b in range(B):
        r = port.select_retained(scores[b].astype(np.float64), d_s)
        np.testing.assert_array_equal(ret[b].cpu().numpy(), r)
        want = port.merge_plan(coords[b], r, k_m)
        dropped = np.setdiff1d(np.arange(N), r)
        np.testing.assert_array_equal(dropped, want["dropped"])
        np.testing.assert_array_equal(tgt[b][dropped], want["target"], err_msg="target")
        assert (tgt[b][r] == -1).all()
        np.testing.assert_array_equal(pcnt[b], want["pool_cnt"], err_msg="pool_cnt")
        np.testing.assert_array_equal(pidx[b], want["pool_idx"], err_msg="pool_idx")
        np.testing.assert_array_equal(pdist[b], want["pool_dist"], err_msg="pool_dist")
        # row_of: retained -> own row, pooled -> pool row, truncated -> -1
        exp_row = np.full(N, -1)
        exp_row[r] = np.arange(len(r))
        for ri in range(len(r)):
            for t in range(want["pool_cnt"][ri]):
                exp_row[want["pool_idx"][ri, t]] = ri
        np.testing.assert_array_equal(row_of[b], exp_row)


@pytest.mark.gpu
@pytest.mark.parametrize("case", PLAN_CASES[:4], ids=[c[0] for c in PLAN_CASES[:4]])
def test_merge_pool_fwd_bwd(case):
    """Values within bf16 tolerance of MergePoolOp (rel-L2 <= 1e-2)."""
    _pool_case(case, 64)


# every compiled row width of the staged pool kernels (16-byte chunks per row 8..64,
# 8 or 16 pool slots) and a width that takes the scalar kernels
POOL_DIMS = [(128, 8), (256, 8), (512, 8), (128, 12), (512, 16), (40, 8)]


@pytest.mark.gpu
@pytest.mark.parametrize("dim,k_m", POOL_DIMS, ids=[f"D{d}_km{k}" for d, k in POOL_DIMS])
def test_merge_pool_dims(dim, k_m):
    _pool_case(("random_dims", lambda rng: random_coords(2, 700, 60.0, rng), 0.3, k_m), dim)


def _pool_case(case, D):
    import torch
    from paper_2602_16249_b200 import ops
    name, mk, d_s, k_m = case
    rng, coords, scores = _plan_problem(name, mk, d_s)
    B, N, _ = coords.shape
    feats = bf16_round(rng.standard_normal((B, N, D)).astype(np.float32))
    p = 1.3
    ret = ops.select_retained(_dev(scores, torch.float32), d_s)
    plan = ops.merge_plan(_dev(coords, torch.float32), ret, k_m)
    fd = _dev(feats, torch.bfloat16)
    sd = _dev(scores, torch.float32)
    pd = _dev([p], torch.float32)
    out = ops.merge_pool_fwd(fd, sd, pd, plan)
    R = ret.shape[1]
    dout = bf16_round(rng.standard_normal((B, R, 2 * D)).astype(np.float32))
    df, ds, dp = ops.merge_pool_bwd(fd, sd, pd, plan, _dev(dout, torch.bfloat16))
    torch.cuda.synchronize()
    out, df, ds, dp = out.float().cpu().numpy(), df.float().cpu().numpy(), ds.cpu().numpy(), float(dp.item())
    want_dp = 0.0
    for b in range(B):
        r = ret[b].cpu().numpy()
        pl = port.merge_plan(coords[b], r, k_m)
        wo = port.merge_pool_fwd(pl, feats[b], scores[b], p)
        assert rel_l2(out[b], wo) <= 1e-2
        wdf, wds, wdp = port.merge_pool_bwd(pl, feats[b], scores[b], p, dout[b])
        assert rel_l2(df[b], wdf) <= 1e-2
        assert rel_l2(ds[b], wds) <= 1e-2
        want_dp += wdp
    assert abs(dp - want_dp) <= 1e-2 * max(1.0, abs(want_dp))
