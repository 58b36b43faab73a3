"""The device-resident training step (csrc/model.cu) against the reference's own Model
(oracle/_ref: proj/src/pipeline.cpp compiled unmodified) on identical inputs:

  * parameter init bit-exact (same splitmix64 draws, pipeline.cpp:255-371);
  * one encode + decode + deep_sup + loss_parts + Tape::backward (pipeline.cpp:402-610,
    tape.cpp:466-724): stage coordinates BIT-EXACT (cluster index, scorer -> select_retained
    -> merge plan -> retained coordinates), loss within 1e-2 relative, stage features and
    every parameter gradient within rel-L2 tolerance of the b32 reference;
  * AdamW steps through train() (pipeline.cpp:682-746): the loss curve follows the
    reference's;
  * checkpoints: the reference's load_checkpoint reads ours, ours reads the reference's
    layout, optimizer state round-trips.

Tolerance.  The device computes bf16 GEMM/attention operands with fp32 accumulation and an
fp32 residual stream; the reference is b32 throughout.  The BASELINE rel-L2 1e-2 bar is met by
the single ops (tests/test_attention_gpu.py, test_merge_gpu.py, ...); a whole network
compounds it, and some gradients are ill-conditioned in the REFERENCE itself: rounding only
its weights to bf16 moves e.g. the merge temperature's or the decoder cross-attention's
gradient by several percent (measured per test case by _sensitivity).  So: stage features
within rel-L2 2e-2; every tensor gradient (norm above 1e-3 of the largest) within
max(5e-2, 5 x the reference's own sensitivity of that tensor to rounding its weights and image
to bf16 -- the device rounds at ~5 places per layer: weights, LN outputs, GEMM outputs,
attention outputs, gradients); the concatenated gradient within max(2e-2, 5 x the overall
sensitivity).  Selection: the retained sets depend
on score ORDER and the device's bf16 scores differ from the b32 reference's by ~1e-3, about
the typical gap between neighbouring scores, so the full-network comparisons teacher-force the
reference's retained sets (Model.force_retained) and test_selection_in_situ pins the device's
own selection bit-exact against the oracle on the scores the device computed.
"""
import numpy as np
import pytest

from oracle import ref
from paper_2602_16249_b200.model import PipelineConfig, StageConfig, step_mask_seed
from tests.problems import rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def small_cfg(**kw):
    st = [StageConfig(64, 2, 2, 16, 3, 0.4, 8), StageConfig(128, 4, 1, 8, 3, 0.4, 8)]
    base = dict(image=64, patch=8, stages=st, dec_dim=64, dec_heads=2, mask_ratio=0.5, batch=1)
    base.update(kw)
    return PipelineConfig(**base)


def tiny_cfg(**kw):
    """AFF-tiny-like at 224^2 with 75% mask (BASELINE configs[0] shape), 3 stages."""
    st = [StageConfig(64, 2, 2, 16, 3, 0.4, 8), StageConfig(128, 4, 2, 16, 3, 0.4, 8),
          StageConfig(256, 8, 2, 16, 3, 0.4, 8)]
    base = dict(image=224, patch=8, stages=st, dec_dim=64, dec_heads=2, mask_ratio=0.75, batch=1)
    base.update(kw)
    return PipelineConfig(**base)


def _models(cfg):
    from paper_2602_16249_b200.model import Model
    mine = Model(cfg)
    theirs = ref.RefModel(cfg.c_struct())
    return mine, theirs


def test_param_table_and_init_bit_exact():
    mine, theirs = _models(small_cfg())
    assert mine.names == theirs.names
    mp, rp = mine.params(), theirs.params()
    for n in mine.names:
        np.testing.assert_array_equal(mp[n].ravel().astype(np.float64), rp[n], err_msg=n)


def _flat(d, names):
    return np.concatenate([np.asarray(d[n], np.float64).ravel() for n in names])


def _sensitivity(cfg, img, mask, tokens, coords):
    """The reference's own gradient change when only its inputs -- the weights and the image,
    the operands the device rounds first -- are rounded to bf16 (rel-L2 per tensor and
    overall): how well-conditioned each gradient is under a 2^-9 relative perturbation."""
    from paper_2602_16249_b200.inputs import bf16_round
    a, b = ref.RefModel(cfg.c_struct()), ref.RefModel(cfg.c_struct())
    b.set_params({n: bf16_round(v.astype(np.float32)).astype(np.float64) for n, v in a.params().items()})
    dims = [st.dim for st in cfg.stages]
    _, ca, _ = a.fwd_bwd(img, mask, tokens, dims)
    _, cb, _ = b.fwd_bwd(bf16_round(img.astype(np.float32)).astype(np.float64), mask, tokens, dims)
    assert all(np.array_equal(x, y) for x, y in zip(ca, cb)), "perturbed reference selects other tokens"
    ga, gb = a.grads(), b.grads()
    return {n: rel_l2(gb[n], ga[n]) for n in ga}, rel_l2(_flat(gb, a.names), _flat(ga, a.names))


def _check_grads(mine, theirs, sens=None, sens_all=0.0, tol_each=5e-2, tol_all=2e-2, factor=5.0):
    """per tensor: rel-L2 <= max(tol_each, factor * the reference's own bf16-weight
    sensitivity of that tensor) for tensors with a non-negligible gradient; overall <=
    max(tol_all, factor * overall sensitivity)."""
    g, w = mine.grads(), theirs.grads()
    norms = {n: np.linalg.norm(w[n]) for n in mine.names}
    big = max(norms.values())
    errs = {n: rel_l2(g[n].ravel(), w[n]) for n in mine.names if norms[n] > 1e-3 * big}
    lim = {n: max(tol_each, factor * (sens or {}).get(n, 0.0)) for n in errs}
    bad = {n: (e, lim[n]) for n, e in errs.items() if e > lim[n]}
    total = rel_l2(_flat(g, mine.names), _flat(w, mine.names))
    return errs, bad, total, max(tol_all, factor * sens_all)


def _retained_from_coords(prev, nxt):
    """indices of the next stage's coordinates inside the previous stage's (lattice points are
    unique, so the reference's retained set is recovered exactly)"""
    at = {(float(x), float(y)): i for i, (x, y) in enumerate(prev)}
    return np.array([at[(float(x), float(y))] for x, y in nxt], np.int32)


def afftiny_full_cfg(**kw):
    """BASELINE configs[0] itself: AFF-tiny 224^2, 4 stages, blocks 3/4/18/5, 75% mask."""
    from paper_2602_16249_b200.model import aff_tiny
    return aff_tiny(batch=1, **kw)


def affmae_b_small_cfg(**kw):
    """The benchmarked AFFMAE-B widths (dims 128/256/512/1024, heads 4/8/16/32, blocks
    3/4/18/2, decoder 256 x 8 heads) on a 128^2 image (64 -> 26 -> 10 -> 4 tokens) so the b32
    reference runs in seconds: every LN / GEMM / attention width of the 1024^2 bench."""
    from paper_2602_16249_b200.model import affmae_b
    return affmae_b(image=128, batch=1, **kw)


def small_depth2_cfg(**kw):
    """two decoder rounds per stage level (DecoderConfig::depth = 2)"""
    return small_cfg(dec_depth=2, **kw)


def small_random_noaux_cfg(**kw):
    """random masks (random_mask, src/masking.cpp:94-110) and no deep supervision (lambda 0)"""
    return small_cfg(mask_strategy="random", lambda_aux=0.0, **kw)


CASES = [(small_cfg, 400), (small_cfg, 412), (tiny_cfg, 408), (tiny_cfg, 411), (afftiny_full_cfg, 402),
         (affmae_b_small_cfg, 403), (small_depth2_cfg, 400), (small_random_noaux_cfg, 401)]


@pytest.mark.parametrize("cfg_fn,img_seed", CASES, ids=[f"{f.__name__[:-4]}_{s}" for f, s in CASES])
def test_forward_backward_matches_reference(cfg_fn, img_seed):
    """Stage coordinates bit-exact, stage features, loss parts and all parameter gradients vs
    the reference.  The merge selection is teacher-forced to the reference's retained sets:
    selection is a discontinuous function of the scores, and the device's bf16 scores differ
    from the b32 reference's by ~1e-3, about the typical gap between neighbouring scores;
    select_retained itself is pinned bit-exact on identical scores (test_merge_gpu.py,
    test_selection_in_situ below)."""
    from paper_2602_16249_b200.model import Model
    cfg = cfg_fn()
    mine, theirs = Model(cfg), ref.RefModel(cfg.c_struct())
    img = ref.synth_image(cfg.image, img_seed)
    seed = step_mask_seed(cfg.seed, 0)
    mask = theirs.make_mask(seed)
    dims = [st.dim for st in cfg.stages]
    want, coords, feats = theirs.fwd_bwd(img, mask, mine.tokens, dims)
    for s in range(len(cfg.stages) - 1):
        mine.force_retained(s, _retained_from_coords(coords[s], coords[s + 1])[None])
    mine.set_images(img[None])
    mine.make_masks([seed])
    np.testing.assert_array_equal(mine.get_masks()[0], mask)
    got = mine.forward_backward()
    for s in range(len(cfg.stages)):
        co, fe, _ = mine.stage_output(s)
        np.testing.assert_array_equal(co[0], coords[s], err_msg=f"stage {s} coordinates")
        e = rel_l2(fe[0], feats[s])
        assert e <= 2e-2, (s, e)
    for a, b, what in zip(got, want, ("total", "main", "aux")):
        assert abs(a - b) <= 1e-2 * abs(b) + 1e-6, (what, a, b)
    sens, sens_all = _sensitivity(cfg, img, mask, mine.tokens, coords)
    errs, bad, total, lim_all = _check_grads(mine, theirs, sens, sens_all)
    assert not bad, f"per-tensor rel-L2 over tolerance (err, limit): {bad}"
    assert total <= lim_all, (total, lim_all, sens_all)


def test_selection_in_situ():
    """Without teacher forcing: every merge keeps exactly select_retained(device scores)
    (the oracle's selection on the scores the device computed) and the next stage's tokens
    are those coordinates, bit-exact."""
    from oracle import port
    from paper_2602_16249_b200.model import Model
    cfg = tiny_cfg(batch=2)
    m = Model(cfg)
    m.set_images(np.stack([ref.synth_image(224, 408), ref.synth_image(224, 409)]))
    m.make_masks([step_mask_seed(1, 0), step_mask_seed(1, 1)])
    m.forward_backward()
    for s in range(len(cfg.stages) - 1):
        co, _, sc = m.stage_output(s)
        nxt, _, _ = m.stage_output(s + 1)
        for b in range(cfg.batch):
            r = port.select_retained(sc[b].astype(np.float64), cfg.stages[s].d_s)
            np.testing.assert_array_equal(nxt[b], co[b][r], err_msg=f"stage {s} image {b}")


def test_batch_is_mean_of_images():
    """B = 2: the gradient of the batch-mean loss equals the mean of the two per-image
    reference gradients (SURVEY §7.4 #7 batch semantics)."""
    from paper_2602_16249_b200.model import Model
    cfg = small_cfg(batch=2)
    mine = Model(cfg)
    imgs = np.stack([ref.synth_image(64, 400), ref.synth_image(64, 402)])
    seeds = [step_mask_seed(1, 0), step_mask_seed(1, 1)]
    mine.set_images(imgs)
    mine.make_masks(seeds)
    acc, losses = None, []
    rets = []
    for b in range(2):
        theirs = ref.RefModel(cfg.c_struct())
        (t, _, _), co, _ = theirs.fwd_bwd(imgs[b], theirs.make_mask(seeds[b]), mine.tokens, [64, 128])
        rets.append(_retained_from_coords(co[0], co[1]))
        losses.append(t)
        w = theirs.grads()
        acc = w if acc is None else {n: acc[n] + w[n] for n in w}
    mine.force_retained(0, np.stack(rets))
    total, _, _ = mine.forward_backward()
    g = mine.grads()
    assert abs(total - np.mean(losses)) <= 1e-2 * abs(np.mean(losses))
    assert rel_l2(_flat(g, mine.names), _flat({n: acc[n] / 2 for n in acc}, mine.names)) <= 2e-2


def test_training_follows_reference_curve():
    """train() for 6 steps on one image (fresh mask per step, AdamW with warmup): the device
    loss curve follows the reference's -- mean relative deviation <= 3e-2, every step within
    0.15 (a step whose selection flips on a near-tie moves by a few percent)."""
    from paper_2602_16249_b200.model import Model
    cfg = small_cfg(warmup=2, total_steps=6, lr=3e-3)
    mine, theirs = Model(cfg), ref.RefModel(cfg.c_struct())
    img = ref.synth_image(64, 403)
    want = theirs.train(6, img[None])
    mine.set_images(img[None])
    got = []
    for step in range(6):
        mine.make_masks([step_mask_seed(cfg.seed, step)])
        got.append(mine.train_step()[0])
    got = np.array(got)
    dev = np.abs(got - want) / np.abs(want)
    assert dev.mean() <= 3e-2 and dev.max() <= 0.15, (got, want)


def test_graph_step_equals_eager_step():
    """The captured CUDA graph of the whole step (forward, backward, AdamW with the step count
    on the device) replays like eager launches: identical first step, and the same trajectory.
    (The reverse-CSR gathers of the decoder backward sum each key's entries in atomic-fill
    order, so later steps agree to fp32 rounding amplified by AdamW's sign-like first updates,
    not bitwise.)"""
    from paper_2602_16249_b200 import devmem
    from paper_2602_16249_b200.model import Model
    cfg = small_cfg(batch=2, warmup=2, total_steps=5)
    imgs = np.stack([ref.synth_image(64, 404), ref.synth_image(64, 405)])
    res = []
    for use_graph in (False, True):
        m = Model(cfg)
        m.set_images(imgs)
        st = devmem.stream_create()
        losses = []
        for step in range(3):
            m.make_masks([step_mask_seed(1, 2 * step), step_mask_seed(1, 2 * step + 1)], stream=st)
            losses.append(m.train_step(use_graph=use_graph, stream=st)[0])
        devmem.sync(st)
        res.append((losses, m.params()))
    (l0, p0), (l1, p1) = res
    assert l0[0] == l1[0]
    np.testing.assert_allclose(l0, l1, rtol=2e-2)
    lr_sum = 1e-3 * (0.5 + 1.0 + 1.0)  # lr_at(0..2) with warmup 2
    for n in p0:
        assert float(np.abs(p0[n] - p1[n]).max()) <= 2 * lr_sum + 1e-6, n


def test_checkpoint_interop(tmp_path):
    """save -> the reference's load_checkpoint reads the parameters (optimizer state lives in
    optim/); load <- restores parameters, moments and the step count."""
    from paper_2602_16249_b200.model import Model
    cfg = small_cfg(warmup=2, total_steps=5)
    m = Model(cfg)
    m.set_images(ref.synth_image(64, 406)[None])
    m.make_masks([step_mask_seed(1, 0)])
    m.train_step()
    d = tmp_path / "ck"
    m.save(str(d))
    got = ref.load_checkpoint(str(d), m.names, [r * c for r, c in m.dims])
    p = m.params()
    for n in m.names:
        np.testing.assert_array_equal(got[n], p[n].ravel().astype(np.float64), err_msg=n)
    m2 = Model(cfg)
    m2.load(str(d))
    p2 = m2.params()
    for n in m.names:
        np.testing.assert_array_equal(p2[n], p[n], err_msg=n)
    # the next step from the restored state equals the uninterrupted one: the updates agree to
    # fp32 rounding (the decoder's parameter-gradient and interpolation reductions use float
    # atomics, so their summation order -- and the last bits -- may vary between two runs)
    m2.set_images(ref.synth_image(64, 406)[None])
    for mm in (m, m2):
        mm.make_masks([step_mask_seed(1, 1)])
        mm.train_step()
    a, b = m.params(), m2.params()
    for n in m.names:
        da, db = (a[n] - p[n]).astype(np.float64), (b[n] - p[n]).astype(np.float64)
        assert np.linalg.norm(db - da) <= 1e-3 * np.linalg.norm(da) + 1e-9, n
