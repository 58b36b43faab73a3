"""Decoder attention over general neighbour rows (one_to_one cross attention, knn self
attention; proj/src/pipeline.cpp:64-71, 495-535) vs the oracle restatement of
nbhd_attn_streaming / nbhd_attn_backward (proj/src/attention.cpp:119-358).

Tolerance as the cluster attention: bf16 inputs, fp32 accumulate,
rel-L2 <= 1e-2 against the b32 oracle on the same bf16-rounded inputs.
"""
import zlib

import numpy as np
import pytest

from oracle import port
from tests.problems import attn_problem, random_coords, rel_l2

REL_TOL = 1e-2


def _nbrs(coords, kind, width, rng):
    """Per-image neighbour rows: 'self' = knn over the image's own tokens (the decoder's
    self_nbr), 'one' = one_to_one, 'holes' = knn with random invalid slots (rows may be
    left with the blank slot only)."""
    B, N, _ = coords.shape
    if kind == "one":
        return np.tile(np.arange(N)[None, :, None], (B, 1, 1)), np.ones((B, N, 1), np.uint8)
    idx, valid = [], []
    for b in range(B):
        i, v = port.knn(coords[b], coords[b], width)
        idx.append(i)
        valid.append(v)
    idx, valid = np.stack(idx), np.stack(valid)
    if kind == "holes":
        valid = valid & (rng.random(valid.shape) < 0.6).astype(np.uint8)
        valid[:, :3] = 0
    return idx, valid


CASES = [  # name, B, N, heads, head_dim, hidden, kind, width
    ("self_dec_default", 2, 700, 4, 16, 8, "self", 8),
    ("cross_one_to_one", 2, 513, 4, 16, 8, "one", 1),
    ("self_holes_d32", 1, 400, 2, 32, 16, "holes", 12),
    ("self_wide_d64", 2, 300, 2, 64, 8, "self", 31),
    ("self_d32_h8", 3, 257, 8, 32, 4, "self", 5),
    ("self_h2_d16", 1, 200, 2, 16, 8, "self", 6),   # 32-wide rows: one dim per lane in the gather
    ("self_h8_d64", 1, 150, 8, 64, 8, "holes", 4),  # 512-wide rows
    ("dec_b_self", 2, 600, 8, 32, 8, "self", 8),    # the AFFMAE-B decoder: 256-wide rows, 8 dims per lane
    ("dec_b_cross", 2, 600, 8, 32, 8, "one", 1),
]


def _problem(case):
    name, B, N, heads, hd, hidden, kind, width = case
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    coords = random_coords(B, N, 224.0, rng)
    pb = attn_problem(coords, heads, hd, hidden, rng)
    pb["idx"], pb["valid"] = _nbrs(coords, kind, width, rng)
    return pb


def _run(pb, gather=True):
    import torch
    from paper_2602_16249_b200 import ops
    dev = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda").contiguous()
    bf = torch.bfloat16
    q, k, v, bk, bv, do = (dev(pb[n], bf) for n in ("q", "k", "v", "bk", "bv", "dout"))
    c = dev(pb["coords"], torch.float32)
    idx, valid = dev(pb["idx"], torch.int32), dev(pb["valid"], torch.uint8)
    bias = ops.BiasNet.from_numpy(pb["bias"])
    out, lse = ops.gattn_fwd(q, k, v, bk, bv, c, idx, valid, bias, pb["heads"], pb["head_dim"])
    g = ops.gattn_bwd(q, k, v, bk, bv, c, idx, valid, bias, pb["heads"], pb["head_dim"], do, gather=gather)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    return f(out), f(lse), {n: f(getattr(g, n)) for n in (
        "dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank")}


def _oracle(pb):
    outs, acc, per = [], None, {"dq": [], "dk": [], "dv": []}
    for b in range(pb["coords"].shape[0]):
        a = (pb["q"][b], pb["k"][b], pb["v"][b], pb["bk"], pb["bv"], pb["coords"][b], pb["idx"][b],
             pb["valid"][b], pb["bias"], pb["heads"], pb["head_dim"])
        outs.append(port.attn_fwd(*a))
        g = port.attn_bwd(*a, pb["dout"][b], prec=32)
        for n in per:
            per[n].append(g[n])
        if acc is None:
            acc = {n: g[n].copy() for n in g if n not in per}
        else:
            for n in acc:
                acc[n] += g[n]
    acc.update({n: np.stack(x) for n, x in per.items()})
    return np.stack(outs), acc


@pytest.mark.gpu
@pytest.mark.parametrize("gather", [True, False], ids=["gather", "scatter"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_gattn_matches_oracle(case, gather):
    pb = _problem(case)
    out, lse, got = _run(pb, gather)
    want_out, want = _oracle(pb)
    assert np.isfinite(out).all() and np.isfinite(lse).all()
    assert rel_l2(out.reshape(want_out.shape), want_out) <= REL_TOL
    report = {n: rel_l2(got[n].reshape(want[n].shape), want[n]) for n in want}
    bad = {n: e for n, e in report.items() if not e <= REL_TOL}
    assert not bad, f"rel-L2 over {REL_TOL}: {bad} (all: {report})"


@pytest.mark.gpu
def test_gattn_lse_and_device_knn():
    """Rows from the device knn (the decoder builds self_nbr with knn, pipeline.cpp:493);
    lse = log sum exp of the row's scores, checked against a float64 numpy restatement."""
    import torch
    from paper_2602_16249_b200 import ops
    case = ("lse", 2, 600, 4, 16, 8, "self", 8)
    pb = _problem(case)
    c = torch.as_tensor(pb["coords"], device="cuda")
    idx, valid = ops.knn(c, c, 8)
    torch.cuda.synchronize()
    assert (idx.cpu().numpy() == pb["idx"]).all() and (valid.cpu().numpy() == pb["valid"]).all()
    _, lse, _ = _run(pb)
    heads, hd, H = 4, 16, 8
    bias = pb["bias"]
    b, i = 1, 77
    q = pb["q"][b, i].reshape(heads, hd).astype(np.float64)
    for h in range(heads):
        s = []
        for j in range(8):
            t = pb["idx"][b, i, j]
            kv = pb["k"][b, t].reshape(heads, hd)[h].astype(np.float64)
            off = (pb["coords"][b, t].astype(np.float64) - pb["coords"][b, i]) / 8.0
            pre = bias["w1"][h, :H] * off[0] + bias["w1"][h, H:] * off[1] + bias["b1"][h]
            s.append(q[h] @ kv / np.sqrt(hd) + bias["b2"].reshape(-1)[h] + bias["w2"][h] @ np.tanh(pre))
        s.append(q[h] @ pb["bk"][h].astype(np.float64) / np.sqrt(hd) + bias["blank"].reshape(-1)[h])
        s = np.array(s)
        want = s.max() + np.log(np.exp(s - s.max()).sum())
        assert abs(lse[b, i, h] - want) < 1e-3


@pytest.mark.gpu
def test_gattn_rejects_bad_width():
    import torch
    from paper_2602_16249_b200 import ops
    pb = _problem(("bad", 1, 64, 2, 16, 4, "self", 8))
    dev = lambda a, dt: torch.as_tensor(a, dtype=dt, device="cuda").contiguous()
    bf = torch.bfloat16
    q = dev(pb["q"], bf)
    idx = torch.zeros((1, 64, 32), dtype=torch.int32, device="cuda")
    valid = torch.ones((1, 64, 32), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="width"):
        ops.gattn_fwd(q, q, q, dev(pb["bk"], bf), dev(pb["bv"], bf), dev(pb["coords"], torch.float32),
                      idx, valid, ops.BiasNet.from_numpy(pb["bias"]), 2, 16)
