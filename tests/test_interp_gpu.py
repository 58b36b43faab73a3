"""Softmax interpolation (make_interp_op, proj/src/interpolation.cpp:192-251) on the GPU
through the C ABI against the oracle restatement (oracle/oracle.c, pinned bit-exact to the
reference by tests/test_oracle_golden.py): outputs and all gradients within rel-L2 1e-2
(bf16 features and cotangents, fp32 arithmetic)."""
import zlib

import numpy as np
import pytest

from oracle import port
from paper_2602_16249_b200.inputs import bf16_round
from tests.problems import lattice_coords, random_coords, rel_l2


def _dev(a, dt):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


# (name, keys, queries, k, dim, p): decoder-like (queries on the full lattice, keys the
# visible tokens), random, coincident query/key, short rows, every compiled width
CASES = [
    ("lattice_dec", lambda r: lattice_coords(2, 64, seed0=7), None, 8, 128, 1.0),
    ("random_d64", lambda r: random_coords(2, 300, 50.0, r), lambda r: random_coords(2, 90, 50.0, r), 6, 64, 1.5),
    ("random_d256", lambda r: random_coords(1, 200, 30.0, r), lambda r: random_coords(1, 70, 30.0, r), 12, 256, 0.7),
    ("k32_d512", lambda r: random_coords(1, 120, 20.0, r), lambda r: random_coords(1, 33, 20.0, r), 32, 512, 2.0),
    ("k1", lambda r: random_coords(2, 40, 10.0, r), lambda r: random_coords(2, 17, 10.0, r), 1, 128, 1.0),
]


@pytest.mark.gpu
@pytest.mark.parametrize("gather", [False, True], ids=["scatter", "gather"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_interp_fwd_bwd(case, gather):
    import torch
    from paper_2602_16249_b200 import ops
    name, mk_keys, mk_q, k, dim, p = case
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    keys = np.ascontiguousarray(mk_keys(rng), np.float32)
    B, N, _ = keys.shape
    if mk_q is None:  # queries: a 2x finer lattice over the same area
        q = np.stack(np.meshgrid(np.arange(64) * 4.0 + 2.0, np.arange(16) * 4.0 + 2.0), -1).reshape(1, -1, 2)
        q = np.repeat(q, B, 0).astype(np.float32)
    else:
        q = np.ascontiguousarray(mk_q(rng), np.float32)
    q[:, 0] = keys[:, 3]  # exact coincidence: zero subgradient
    Q = q.shape[1]
    idx, valid = ops.knn(_dev(q, torch.float32), _dev(keys, torch.float32), k)
    if k > 2:
        valid[:, 1, k // 2:] = 0  # a short row
    feats = bf16_round(rng.standard_normal((B, N, dim)).astype(np.float32))
    dout = bf16_round(rng.standard_normal((B, Q, dim)).astype(np.float32))
    pd = _dev([p], torch.float32)
    qd, kd = _dev(q, torch.float32), _dev(keys, torch.float32)
    fd = _dev(feats, torch.bfloat16)
    out = ops.interp_fwd(qd, kd, fd, idx, valid, pd)
    df, dp, dq = ops.interp_bwd(qd, kd, fd, idx, valid, pd, _dev(dout, torch.bfloat16), gather=gather)
    torch.cuda.synchronize()
    out, df, dq, dp = out.float().cpu().numpy(), df.cpu().numpy(), dq.cpu().numpy(), float(dp.item())
    ii, vv = idx.cpu().numpy(), valid.cpu().numpy()
    want_dp = 0.0
    for b in range(B):
        wo = port.interp_fwd(q[b], keys[b], feats[b], ii[b], vv[b], p)
        assert rel_l2(out[b], wo) <= 1e-2, name
        wdf, wdp, wdq = port.interp_bwd(q[b], keys[b], feats[b], ii[b], vv[b], p, dout[b])
        assert rel_l2(df[b], wdf) <= 1e-2
        assert rel_l2(dq[b], wdq) <= 1e-2
        assert dq[b, 0, 0] == dq[b, 0, 0]  # finite at the coincidence
        want_dp += wdp
    assert abs(dp - want_dp) <= 1e-2 * max(1.0, abs(want_dp))


@pytest.mark.gpu
def test_interp_bwd_gather_accumulates_like_scatter():
    """The reverse-CSR backward adds into existing gradients (CustomOp +=) and matches the
    scattered-reduction backward to fp32 rounding, at the decoder's size class."""
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(3)
    keys = _dev(lattice_coords(3, 64, seed0=11), torch.float32)
    g = np.stack(np.meshgrid(np.arange(64) * 8.0 + 4.0, np.arange(64) * 8.0 + 4.0), -1).reshape(1, -1, 2)
    q = _dev(np.repeat(g, 3, 0).astype(np.float32), torch.float32)
    feats = _dev(rng.standard_normal((3, keys.shape[1], 128)), torch.bfloat16)
    dout = _dev(rng.standard_normal((3, q.shape[1], 128)), torch.bfloat16)
    pd = _dev([1.3], torch.float32)
    idx, valid = ops.knn(q, keys, 8)
    res = []
    for gather in (False, True):
        df = torch.ones((3, keys.shape[1], 128), dtype=torch.float32, device="cuda")
        dp = torch.full((1,), 0.5, device="cuda")
        dq = torch.ones((3, q.shape[1], 2), device="cuda")
        ops.interp_bwd(q, keys, feats, idx, valid, pd, dout, dfeats=df, dp=dp, dqueries=dq, gather=gather)
        res.append((df.cpu().numpy(), float(dp.item()), dq.cpu().numpy()))
    (a, ap, aq), (b, bp, bq) = res
    assert np.abs(a - b).max() <= 1e-4 * max(1.0, np.abs(a).max())
    assert abs(ap - bp) <= 1e-4 * max(1.0, abs(ap)) and np.array_equal(aq, bq)


@pytest.mark.gpu
def test_interp_rejects_unsupported():
    import torch
    from paper_2602_16249_b200 import ops
    z = torch.zeros((1, 4, 2), dtype=torch.float32, device="cuda")
    f = torch.zeros((1, 4, 40), dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros((1, 4, 2), dtype=torch.int32, device="cuda")
    val = torch.ones((1, 4, 2), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):  # ConfigError taxonomy: dim 40 not compiled
        ops.interp_fwd(z, z, f, idx, val, torch.ones(1, device="cuda"))
    with pytest.raises(ValueError):  # K > 32
        big = torch.zeros((1, 4, 33), dtype=torch.int32, device="cuda")
        ops.interp_fwd(z, z, torch.zeros((1, 4, 64), dtype=torch.bfloat16, device="cuda"), big,
                       torch.ones((1, 4, 33), dtype=torch.uint8, device="cuda"), torch.ones(1, device="cuda"))


@pytest.mark.gpu
@pytest.mark.parametrize("gather", [False, True], ids=["scatter", "gather"])
def test_interp_bwd_empty_rows_and_unreferenced_keys(gather):
    """A row with no valid neighbour contributes nothing, keys no row names keep their
    accumulated gradient untouched (+= semantics), in both backward forms."""
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(17)
    keys = _dev(random_coords(1, 64, 40.0, rng), torch.float32)
    q = _dev(random_coords(1, 20, 10.0, rng), torch.float32)  # a corner: far keys unreferenced
    feats = _dev(rng.standard_normal((1, 64, 64)), torch.bfloat16)
    dout = _dev(rng.standard_normal((1, 20, 64)), torch.bfloat16)
    idx, valid = ops.knn(q, keys, 4)
    valid[0, 5] = 0  # an empty row
    pd = _dev([1.0], torch.float32)
    df = torch.full((1, 64, 64), 0.25, device="cuda")
    dq = torch.zeros((1, 20, 2), device="cuda")
    ops.interp_bwd(q, keys, feats, idx, valid, pd, dout, dfeats=df, dqueries=dq, gather=gather)
    out = ops.interp_fwd(q, keys, feats, idx, valid, pd)
    torch.cuda.synchronize()
    named = set(idx[valid.bool()].cpu().numpy().tolist())
    untouched = [j for j in range(64) if j not in named]
    assert untouched and (df[0, untouched] == 0.25).all()
    assert (dq[0, 5] == 0).all() and (out[0, 5].float() == 0).all()
