"""Dense linear layer on tcgen05 (the Tape's matmul + bias + gelu_erf,
proj/src/tape.cpp / proj/src/pipeline.cpp:388-400) against a plain PyTorch fp32 reference of
the same op on the same bf16-rounded inputs: rel-L2 <= 1e-2."""
import pytest


def _rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,act", [(4096, 384, 128, "none"),   # QKV projection, D = 128
                                       (4096, 512, 128, "gelu"),   # MLP fc1 (4D), GELU(erf)
                                       (4096, 128, 512, "none"),   # MLP fc2
                                       (1000, 136, 264, "gelu"),   # ragged M, N, K (multiples of 8)
                                       (1, 64, 8, "none")])
def test_linear_matches_fp32_reference(m, n, k, act):
    import torch
    from paper_2602_16249_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    x = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((n, k), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    b = torch.randn(n, device="cuda", generator=g)
    y = ops.linear(x, w, b, act=act).float()
    ref = x.float() @ w.float().t() + b
    if act == "gelu":
        ref = torch.nn.functional.gelu(ref)  # erf form, as the reference's gelu_erf
    assert _rel(y, ref) <= 1e-2


@pytest.mark.gpu
def test_linear_rejects_unaligned():
    import torch
    from paper_2602_16249_b200 import ops
    x = torch.zeros((16, 12), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((8, 12), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        ops.linear(x, w)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [(4096, 512, 128), (4096, 128, 512), (1000, 136, 264)])
def test_linear_backward_matches_fp32_reference(m, n, k):
    import torch
    from paper_2602_16249_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(m * 3 + n + k)
    x = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((n, k), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    dy = torch.randn((m, n), device="cuda", generator=g).to(torch.bfloat16)
    dw0 = torch.randn((n, k), device="cuda", generator=g)
    db0 = torch.randn(n, device="cuda", generator=g)
    dx, dw, db = ops.linear_bwd(x, w, dy, dw=dw0.clone(), db=db0.clone())
    assert _rel(dx.float(), dy.float() @ w.float()) <= 1e-2
    assert _rel(dw, dw0 + dy.float().t() @ x.float()) <= 1e-2  # accumulated (+=)
    assert _rel(db, db0 + dy.float().sum(0)) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(4096, 128), (3000, 256), (1000, 384), (777, 1024), (1, 512)])
def test_layer_norm_matches_fp32_reference(rows, cols):
    """Tape::layer_norm and its VJP (proj/src/tape.cpp:84-100,581-617, eps 1e-5)."""
    import torch
    from paper_2602_16249_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    x = (torch.randn((rows, cols), device="cuda", generator=g) * 3 + 1).to(torch.bfloat16)
    gamma = torch.randn(cols, device="cuda", generator=g)
    beta = torch.randn(cols, device="cuda", generator=g)
    dy = torch.randn((rows, cols), device="cuda", generator=g).to(torch.bfloat16)
    y, stats = ops.layer_norm(x, gamma, beta)
    xf = x.float().requires_grad_(True)
    gf, bf = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xf, (cols,), gf, bf, eps=1e-5)
    assert _rel(y.float(), ref.detach()) <= 1e-2
    ref.backward(dy.float())
    dg0, db0 = torch.ones(cols, device="cuda"), torch.ones(cols, device="cuda")
    dx, dg, db = ops.layer_norm_bwd(x, gamma, stats, dy, dgamma=dg0.clone(), dbeta=db0.clone())
    assert _rel(dx.float(), xf.grad) <= 1e-2
    assert _rel(dg, dg0 + gf.grad) <= 1e-3 and _rel(db, db0 + bf.grad) <= 1e-3


@pytest.mark.gpu
def test_mlp_block_fwd_bwd_matches_fp32_reference():
    """fc1 + GELU (pre-activation saved) -> fc2, and the whole backward on the GPU ops, vs torch
    autograd in fp32 on the same bf16 inputs."""
    import torch
    from paper_2602_16249_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(11)
    M, D = 2048, 128
    x = torch.randn((M, D), device="cuda", generator=g).to(torch.bfloat16)
    w1 = (torch.randn((4 * D, D), device="cuda", generator=g) / D ** 0.5).to(torch.bfloat16)
    b1 = torch.randn(4 * D, device="cuda", generator=g) * 0.1
    w2 = (torch.randn((D, 4 * D), device="cuda", generator=g) / (4 * D) ** 0.5).to(torch.bfloat16)
    b2 = torch.randn(D, device="cuda", generator=g) * 0.1
    dy = torch.randn((M, D), device="cuda", generator=g).to(torch.bfloat16)
    h, pre = ops.linear_gelu_save(x, w1, b1)
    y = ops.linear(h, w2, b2)
    dh, dw2, db2 = ops.linear_bwd(h, w2, dy)
    dpre = ops.gelu_bwd(pre, dh)
    dx, dw1, db1 = ops.linear_bwd(x, w1, dpre)
    xf = x.float().requires_grad_(True)
    w1f, b1f = w1.float().requires_grad_(True), b1.clone().requires_grad_(True)
    w2f, b2f = w2.float().requires_grad_(True), b2.clone().requires_grad_(True)
    pref = xf @ w1f.t() + b1f
    yf = torch.nn.functional.gelu(pref) @ w2f.t() + b2f
    yf.backward(dy.float())
    assert _rel(pre.float(), pref.detach()) <= 1e-2
    assert _rel(y.float(), yf.detach()) <= 1e-2
    for got, want in ((dx, xf.grad), (dw1, w1f.grad), (db1, b1f.grad), (dw2, w2f.grad), (db2, b2f.grad)):
        assert _rel(got.float(), want) <= 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [(262144, 384, 128),   # stage-0 QKV of the AFFMAE-B step (64 images)
                                   (41920, 2048, 512),   # stage-2 MLP fc1
                                   (16768, 1024, 4096),  # stage-3 MLP fc2
                                   (2050, 16, 256),      # merge scorer (N = 16: one 64-wide tile, masked)
                                   (65536, 136, 64),     # split dW with the fused bias sums, ragged M tile
                                   (4100, 512, 520),     # CTA-pair forward with a K tail and a ragged M tile
                                   (300, 72, 40)])       # ragged everything
def test_linear_step_shapes(m, n, k):
    """The training step's GEMM shapes on the hand-written tcgen05 kernel (gemm_tc.cu): forward
    (K-major operands), dX (N-major W), dW over every token (M- and N-major operands, split-K
    partials reduced in a fixed order, the bias gradient from the operand ring when split >= 8
    ways) against torch fp32."""
    import torch
    from paper_2602_16249_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(m + 7 * n + k)
    x = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((n, k), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    b = torch.randn(n, device="cuda", generator=g)
    dy = torch.randn((m, n), device="cuda", generator=g).to(torch.bfloat16)
    y = ops.linear(x, w, b).float()
    assert _rel(y, x.float() @ w.float().t() + b) <= 1e-2
    dw0 = torch.randn((n, k), device="cuda", generator=g)
    dx, dw, db = ops.linear_bwd(x, w, dy, dw=dw0.clone())
    assert _rel(dx.float(), dy.float() @ w.float()) <= 1e-2
    assert _rel(dw - dw0, dy.float().t() @ x.float()) <= 1e-2
    assert _rel(db, dy.float().sum(0)) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("m,d", [(8192, 128), (1000, 256), (4100, 512)])
def test_linear_fused_epilogues(m, d):
    """GELU-aux forward, residual-add forward, dX with the GELU derivative fused, and the fp32
    dX with beta (the model's residual-stream gradient accumulation) against torch fp32."""
    import torch
    from paper_2602_16249_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(m + d)
    x = torch.randn((m, d), device="cuda", generator=g).to(torch.bfloat16)
    w1 = (torch.randn((4 * d, d), device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    b1 = torch.randn(4 * d, device="cuda", generator=g) * 0.1
    w2 = (torch.randn((d, 4 * d), device="cuda", generator=g) / (4 * d) ** 0.5).to(torch.bfloat16)
    b2 = torch.randn(d, device="cuda", generator=g) * 0.1
    c = torch.randn((m, d), device="cuda", generator=g).to(torch.bfloat16)
    h, pre = ops.linear_gelu_save(x, w1, b1)
    pref = x.float() @ w1.float().t() + b1
    assert _rel(pre.float(), pref) <= 1e-2
    assert _rel(h.float(), torch.nn.functional.gelu(pre.float())) <= 1e-2
    y = ops.linear_add(h, w2, b2, c)
    assert _rel(y.float(), h.float() @ w2.float().t() + b2 + c.float()) <= 1e-2
    dy = torch.randn((m, d), device="cuda", generator=g).to(torch.bfloat16)
    dh = ops.linear_dx_gelu(dy, w2, pre)
    pf = pre.float()
    gp = 0.5 * (1 + torch.erf(pf / 2 ** 0.5)) + pf * torch.exp(-0.5 * pf * pf) / (2 * torch.pi) ** 0.5
    assert _rel(dh.float(), (dy.float() @ w2.float()) * gp) <= 1e-2
    dx0 = torch.randn((m, 4 * d), device="cuda", generator=g)
    dx = ops.linear_dx_f32(dy, w2, dx=dx0.clone(), beta=1.0)
    assert _rel(dx, dx0 + dy.float() @ w2.float()) <= 1e-3
    dx = ops.linear_dx_f32(dy, w2, dx=dx0.clone(), beta=0.0)
    assert _rel(dx, dy.float() @ w2.float()) <= 1e-3
