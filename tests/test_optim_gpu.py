"""Fused AdamW (AdamW::step, proj/src/pipeline.cpp:639-680) on the GPU through the C ABI
against the oracle restatement (pinned bit-exact to the reference by
tests/test_oracle_golden.py::test_adamw_matches_reference).  The device keeps the moments
in fp32 (the reference in binary64), so values agree to fp32 rounding, not bitwise."""
import numpy as np
import pytest

from oracle import port


@pytest.mark.gpu
@pytest.mark.parametrize("warmup,total,steps", [(3, 10, 8), (100, 1000, 5), (1, 2, 4)])
def test_adamw_matches_oracle(warmup, total, steps):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(warmup * 7 + total)
    shapes = [(64, 33), (1, 33), (5, 7, 3), (1, 1), (129,), (2, 2)]
    opt = ops.AdamW(shapes, lr=2e-3, warmup=warmup, total_steps=total)
    flat = [rng.standard_normal(int(np.prod(s))).astype(np.float32) for s in shapes]
    for p, v in zip(opt.params, flat):
        p.copy_(torch.as_tensor(v.reshape(p.shape)))
    grads = [[(rng.standard_normal(int(np.prod(s))) * 0.1).astype(np.float32) for s in shapes] for _ in range(steps)]
    for st in range(steps):
        for g, v in zip(opt.grads, grads[st]):
            g.copy_(torch.as_tensor(v.reshape(g.shape)))
        opt.step()
        assert abs(opt.lr_at(st) - port.lib().orc_adamw_lr(2e-3, warmup, total, st)) == 0.0
    torch.cuda.synchronize()
    got = np.concatenate([p.cpu().numpy().reshape(-1) for p in opt.params])
    # the oracle's decay rule is on the 2-D view (rows = dim(0)), as the reference's Tensor
    oshapes = [(s[0], int(np.prod(s[1:])) if len(s) > 1 else 1) for s in shapes]
    want, _, _ = port.adamw(oshapes, np.concatenate(flat), np.stack([np.concatenate(g) for g in grads]),
                            lr=2e-3, warmup=warmup, total=total)
    np.testing.assert_allclose(got, want, rtol=2e-5, atol=2e-6)


@pytest.mark.gpu
def test_adamw_rejects_bad_config():
    from paper_2602_16249_b200 import ops
    opt = ops.AdamW([(2, 2)], total_steps=0)
    with pytest.raises(ValueError):
        opt.step()
