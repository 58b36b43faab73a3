"""The merge's standalone functions against the compiled reference (oracle/_ref):
importance_scores (proj/src/merging.cpp:31-48; binary64 in the reference's order, so equal to
the b32 output up to the last bit of the device erf / exp) and merge_tokens with its
layer_norm_rows (proj/src/merging.cpp:222-273; plan and retained coordinates bit-exact, merged
features within rel-L2 1e-2 of the b32 reference on the same bf16 inputs)."""
import numpy as np
import pytest

from oracle import ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _dev(a, dtype):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _bf16_round(a):
    import torch
    return torch.as_tensor(np.asarray(a, np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


@pytest.mark.parametrize("n,d,h", [(1000, 64, 8), (777, 128, 16), (300, 512, 32), (64, 1024, 5)])
def test_importance_scores_matches_reference(n, d, h):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(n + d + h)
    f = rng.standard_normal((n, d)).astype(np.float32)
    w1 = (rng.standard_normal((d, h)) / np.sqrt(d)).astype(np.float32)
    b1 = (0.1 * rng.standard_normal(h)).astype(np.float32)
    w2 = rng.standard_normal(h).astype(np.float32)
    b2 = np.float32(0.05)
    got = ops.importance_scores(_dev(f, torch.float32), _dev(w1, torch.float32), _dev(b1, torch.float32),
                                _dev(w2, torch.float32), _dev([b2], torch.float32)).cpu().numpy()
    want = ref.importance_scores(f, w1, b1, w2, float(b2), prec=32)
    np.testing.assert_allclose(got, want.astype(np.float32), rtol=2.5e-7, atol=0)


def _lattice(n, side, rng):
    cells = rng.choice(side * side, n, replace=False)
    return np.stack([(cells % side) * 8 + 4, (cells // side) * 8 + 4], 1).astype(np.float32)


@pytest.mark.parametrize("kind,n,d,k_m,p", [("lattice", 600, 64, 8, 1.0), ("random", 900, 128, 8, 1.5),
                                            ("lattice", 1500, 256, 4, 1.0)])
def test_merge_tokens_matches_reference(kind, n, d, k_m, p):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(n + d)
    B = 2
    coords = np.stack([_lattice(n, 64, rng) if kind == "lattice" else rng.uniform(0, 400, (n, 2)).astype(np.float32)
                       for _ in range(B)])
    feats = _bf16_round(rng.standard_normal((B, n, d)))
    scores = rng.uniform(0.1, 0.9, (B, n)).astype(np.float32)
    r = ref.retained_count(n, 0.4)
    retained = np.stack([np.sort(rng.choice(n, r, replace=False)) for _ in range(B)]).astype(np.int32)
    proj_w = _bf16_round(rng.standard_normal((2 * d, d)) / np.sqrt(2 * d))
    gamma = (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(d)).astype(np.float32)
    oc, of = ops.merge_tokens(_dev(coords, torch.float32), _dev(feats, torch.bfloat16), _dev(scores, torch.float32),
                              _dev(retained, torch.int32), k_m, _dev([p], torch.float32),
                              _dev(proj_w.T, torch.bfloat16), _dev(gamma, torch.float32), _dev(beta, torch.float32))
    oc, of = oc.cpu().numpy(), of.float().cpu().numpy()
    for b in range(B):
        wc, wf = ref.merge_tokens(coords[b], feats[b], scores[b], retained[b], k_m, p, proj_w, gamma, beta, prec=32)
        np.testing.assert_array_equal(oc[b], wc.astype(np.float32))
        rel = np.linalg.norm(of[b] - wf) / np.linalg.norm(wf)
        assert rel <= 1e-2, (b, rel)


def test_merge_tokens_all_retained_and_single_contributor():
    """d_s = 1 (every token retained: pools hold only the empty aggregate) and k_m = 1."""
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(7)
    n, d = 200, 64
    coords = _lattice(n, 32, rng)[None]
    feats = _bf16_round(rng.standard_normal((1, n, d)))
    scores = rng.uniform(0.1, 0.9, (1, n)).astype(np.float32)
    proj_w = _bf16_round(rng.standard_normal((2 * d, d)) / np.sqrt(2 * d))
    gamma, beta = np.ones(d, np.float32), np.zeros(d, np.float32)
    for retained, k_m in ((np.arange(n), 8), (np.sort(rng.choice(n, 80, replace=False)), 1)):
        retained = retained.astype(np.int32)[None]
        oc, of = ops.merge_tokens(_dev(coords, torch.float32), _dev(feats, torch.bfloat16),
                                  _dev(scores, torch.float32), _dev(retained, torch.int32), k_m,
                                  _dev([1.0], torch.float32), _dev(proj_w.T, torch.bfloat16),
                                  _dev(gamma, torch.float32), _dev(beta, torch.float32))
        wc, wf = ref.merge_tokens(coords[0], feats[0], scores[0], retained[0], k_m, 1.0, proj_w, gamma, beta)
        np.testing.assert_array_equal(oc.cpu().numpy()[0], wc.astype(np.float32))
        got = of.float().cpu().numpy()[0]
        assert np.linalg.norm(got - wf) / np.linalg.norm(wf) <= 1e-2


def test_importance_scores_rejects_mismatched_width():
    import torch
    from paper_2602_16249_b200 import ops
    f = torch.zeros((4, 32), dtype=torch.float32, device="cuda")
    w1 = torch.zeros((16, 8), dtype=torch.float32, device="cuda")
    z = torch.zeros(8, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match="feature width"):
        ops.importance_scores(f, w1, z, z, z[:1])
