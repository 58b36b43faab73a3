"""Small-shape run of every hand-written kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck / initcheck).  Usage (GPU box):

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool racecheck \
        python tools/sanitize_probe.py

Shapes are chosen to reach the interesting code paths while staying small:
the clustered DSMEM segment sort (several images over CTA clusters), the lattice
fast and general attention kernels (cp.async rings, the bias-table RMW and its
duplicate-coordinate atomic fallback), the radix select, merge plan and the
staged pool kernels, masks, interpolation and decoder attention.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16249_b200 import inputs, ops  # noqa: E402


def dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def attn_round(coords, heads, hd, rng):
    B, N, _ = coords.shape
    bf = torch.bfloat16
    r = lambda *s: dev(0.5 * rng.standard_normal(s), bf)
    q, k, v, bk, bv = r(B, N, heads * hd), r(B, N, heads * hd), r(B, N, heads * hd), r(heads, hd), r(heads, hd)
    c = dev(coords, torch.float32)
    geom = ops.geometry(B, N, 16, 3)
    index = ops.cluster_index(c, 16, 3)
    bias = ops.BiasNet.from_numpy(inputs.bias_params(heads, 8, rng))
    plan = ops.attn_plan(geom, c, index, heads, hd, 8)
    o, l = ops.attn_fwd(geom, q, k, v, bk, bv, c, None, None, bias, heads, hd, plan=plan)
    ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, heads, hd, o, l, r(B, N, heads * hd), plan=plan)
    torch.cuda.synchronize()


def main():
    rng = np.random.default_rng(0)
    which = sys.argv[1:] or ["index", "attn", "merge", "masks", "decoder", "model"]
    lat = inputs.lattice_batch(3, 48, 0.75, 8, 1000)  # N = 576, 3 images
    if "index" in which:
        ops.cluster_index(dev(lat, torch.float32), 16, 3)
        ops.cluster_index(dev(rng.uniform(0, 300, (6, 3000, 2)), torch.float32), 16, 3)
        ops.knn(dev(rng.uniform(0, 50, (2, 1500, 2)), torch.float32),
                dev(rng.uniform(0, 50, (2, 800, 2)), torch.float32), 8)
        torch.cuda.synchronize()
        print("index ok", flush=True)
    if "attn" in which:
        attn_round(lat, 4, 32, rng)
        attn_round(rng.uniform(0, 120, (2, 400, 2)).astype(np.float32), 2, 32, rng)
        dup = lat.copy()
        dup[:, 1::2] = dup[:, 0::2]
        attn_round(dup, 2, 32, rng)
        print("attention ok", flush=True)
    if "merge" in which:
        n = lat.shape[1]
        s = dev(rng.uniform(0.1, 0.9, (3, n)), torch.float32)
        ret = ops.select_retained(s, 0.4)
        plan = ops.merge_plan(dev(lat, torch.float32), ret, 8)
        f = dev(rng.standard_normal((3, n, 128)), torch.bfloat16)
        p = dev([1.0], torch.float32)
        out = ops.merge_pool_fwd(f, s, p, plan)
        ops.merge_pool_bwd(f, s, p, plan, torch.randn_like(out))
        torch.cuda.synchronize()
        print("merge ok", flush=True)
    if "masks" in which:
        m = ops.perlin_masks([11, 12], 40, 0.75)
        ops.visible_coords(m)
        ops.synth_images([400, 401], 64)
        torch.cuda.synchronize()
        print("masks ok", flush=True)
    if "decoder" in which:
        keys = dev(lat, torch.float32)
        qs = dev(rng.uniform(0, 384, (3, 300, 2)), torch.float32)
        idx, valid = ops.knn(qs, keys, 8)
        f = dev(rng.standard_normal((3, lat.shape[1], 128)), torch.bfloat16)
        p = dev([1.0], torch.float32)
        out = ops.interp_fwd(qs, keys, f, idx, valid, p)
        ops.interp_bwd(qs, keys, f, idx, valid, p, torch.randn_like(out))
        # decoder attention at the AFFMAE-B row width (8 heads x 32): the register row forward
        # (8-wide knn rows), the shared-memory-staged row kernels (one-to-one rows), the thread
        # backward with the reverse-CSR gather
        heads, hd, n = 8, 32, 300
        c = dev(rng.uniform(0, 200, (2, n, 2)), torch.float32)
        r = lambda *sh: dev(0.5 * rng.standard_normal(sh), torch.bfloat16)
        q, k, v, bk, bv = r(2, n, heads * hd), r(2, n, heads * hd), r(2, n, heads * hd), r(heads, hd), r(heads, hd)
        bias = ops.BiasNet.from_numpy(inputs.bias_params(heads, 8, rng))
        si, sv = ops.knn(c, c, 8)
        oi = torch.arange(n, dtype=torch.int32, device="cuda").repeat(2, 1).reshape(2, n, 1).contiguous()
        ov = torch.ones(2, n, 1, dtype=torch.uint8, device="cuda")
        for ii, vv in ((si, sv), (oi, ov)):
            o, _ = ops.gattn_fwd(q, k, v, bk, bv, c, ii, vv, bias, heads, hd)
            ops.gattn_bwd(q, k, v, bk, bv, c, ii, vv, bias, heads, hd, torch.randn_like(o), gather=True,
                          workspace=torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
            ops.gattn_bwd(q, k, v, bk, bv, c, ii, vv, bias, heads, hd, torch.randn_like(o))
        torch.cuda.synchronize()
        print("decoder ok", flush=True)
    if "model" in which:
        model_round()
        print("model ok", flush=True)


def model_round():
    """one training step of a small two-stage model: every model kernel (row LN fwd/bwd, pos
    MLP, scorer, offset head, gathers, bias column sums, AdamW with the device step)"""
    from paper_2602_16249_b200.model import Model, PipelineConfig, StageConfig, step_mask_seed
    st = [StageConfig(64, 2, 2, 16, 3, 0.4, 8), StageConfig(128, 4, 1, 8, 3, 0.4, 8)]
    m = Model(PipelineConfig(image=64, patch=8, stages=st, dec_dim=64, dec_heads=2, mask_ratio=0.5, batch=2))
    rng = np.random.default_rng(1)
    m.set_images(rng.uniform(0, 1, (2, 64, 64)))
    m.make_masks([step_mask_seed(1, 0), step_mask_seed(1, 1)])
    m.train_step()
    m.close()


if __name__ == "__main__":
    main()
