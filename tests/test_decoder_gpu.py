"""Decoder row ops on the GPU against plain fp32 restatements of the
reference: NormClampOp (proj/src/pipeline.cpp:75-127) and the masked reconstruction loss
(Tape::mse, proj/src/tape.cpp:431-446,694-707)."""
import numpy as np
import pytest


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("rows,d,limit", [(2000, 64, 1.0), (700, 100, 5.0), (1, 33, 0.1)])
def test_norm_clamp_fwd_bwd(rows, d, limit):
    import torch
    from paper_2602_16249_b200 import ops
    from paper_2602_16249_b200.inputs import bf16_round
    rng = np.random.default_rng(rows + d)
    x = bf16_round((rng.standard_normal((rows, d)) * rng.uniform(0.01, 3.0, (rows, 1))).astype(np.float32))
    g = bf16_round(rng.standard_normal((rows, d)).astype(np.float32))
    y = ops.norm_clamp(torch.as_tensor(x, device="cuda").to(torch.bfloat16), limit).float().cpu().numpy()
    dx = ops.norm_clamp_bwd(torch.as_tensor(x, device="cuda").to(torch.bfloat16),
                            torch.as_tensor(g, device="cuda").to(torch.bfloat16), limit).float().cpu().numpy()
    x64, g64 = x.astype(np.float64), g.astype(np.float64)
    r = np.sqrt((x64 ** 2).sum(1, keepdims=True))
    f = np.where(r > limit, limit / np.maximum(r, 1e-300), 1.0)
    assert _rel(y, x64 * f) <= 1e-2
    dot = (g64 * x64).sum(1, keepdims=True) / np.maximum(r * r, 1e-300)
    want = np.where(r <= limit, g64, f * (g64 - dot * x64))
    assert _rel(dx, want) <= 1e-2
    # CustomOp::backward semantics: a second call accumulates into the same dx
    base = bf16_round(rng.standard_normal((rows, d)).astype(np.float32))
    acc = torch.as_tensor(base, device="cuda").to(torch.bfloat16)
    ops.norm_clamp_bwd(torch.as_tensor(x, device="cuda").to(torch.bfloat16),
                       torch.as_tensor(g, device="cuda").to(torch.bfloat16), limit, dx=acc)
    assert _rel(acc.float().cpu().numpy(), base + want) <= 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("rows,p,cells", [(12288, 64, 16384), (100, 48, 300), (1, 64, 1)])
def test_masked_mse(rows, p, cells):
    import torch
    from paper_2602_16249_b200 import ops
    from paper_2602_16249_b200.inputs import bf16_round
    rng = np.random.default_rng(rows * 7 + p)
    patches = rng.standard_normal((cells, p)).astype(np.float32)
    idx = np.sort(rng.choice(cells, rows, replace=False)).astype(np.int32)
    pred = bf16_round(rng.standard_normal((rows, p)).astype(np.float32))
    loss, dpred = ops.masked_mse(torch.as_tensor(pred, device="cuda").to(torch.bfloat16),
                                 torch.as_tensor(patches, device="cuda"), torch.as_tensor(idx, device="cuda"),
                                 dloss=0.5)
    diff = pred.astype(np.float64) - patches[idx].astype(np.float64)
    assert abs(float(loss.item()) - (diff ** 2).mean()) <= 1e-4 * max(1.0, (diff ** 2).mean())
    assert _rel(dpred.float().cpu().numpy(), 0.5 * 2.0 * diff / diff.size) <= 1e-2
