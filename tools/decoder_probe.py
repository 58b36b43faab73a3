"""Decoder-shape micro-benchmarks for the training step (B200): decoder self-attention backward
(scattered vs reverse-CSR gather), the MLP fc1 GEMM with the fused GELU epilogue vs GEMM + a
separate GELU pass, knn over a sparse stage.

    python tools/decoder_probe.py [--batch 16]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16249_b200 import inputs, ops  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    a = ap.parse_args()
    B, g = a.batch, 128
    rng = np.random.default_rng(0)
    masks = ops.perlin_masks(list(range(B)), g, 0.75)
    refs, _ = ops.visible_coords(1 - masks)  # masked cells = the decoder's queries
    Q = refs.shape[1]
    heads, hd, hidden = 8, 32, 8
    D = heads * hd
    idx, valid = ops.knn(refs, refs, 8)
    bf = torch.bfloat16
    t = lambda *s: torch.randn(*s, device="cuda").to(bf) * 0.5
    q, k, v, bk, bv = t(B, Q, D), t(B, Q, D), t(B, Q, D), t(heads, hd), t(heads, hd)
    bias = ops.BiasNet.from_numpy(inputs.bias_params(heads, hidden, rng))
    out, lse = ops.gattn_fwd(q, k, v, bk, bv, refs, idx, valid, bias, heads, hd)
    dout = t(B, Q, D)
    print(f"B={B} Q={Q} tokens={B * Q}")
    print("gattn fwd            %.3f ms" % timeit(lambda: ops.gattn_fwd(q, k, v, bk, bv, refs, idx, valid, bias, heads, hd)))
    print("gattn bwd scatter    %.3f ms" % timeit(lambda: ops.gattn_bwd(q, k, v, bk, bv, refs, idx, valid, bias, heads, hd,
                                                                    dout)))
    ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    print("gattn bwd gather     %.3f ms" % timeit(lambda: ops.gattn_bwd(q, k, v, bk, bv, refs, idx, valid, bias, heads, hd,
                                                                    dout, gather=True, workspace=ws)))
    i1 = torch.arange(Q, dtype=torch.int32, device="cuda").repeat(B, 1).reshape(B, Q, 1).contiguous()
    v1 = torch.ones(B, Q, 1, dtype=torch.uint8, device="cuda")
    print("gattn cross fwd      %.3f ms" % timeit(lambda: ops.gattn_fwd(q, k, v, bk, bv, refs, i1, v1, bias, heads, hd)))
    print("gattn cross bwd      %.3f ms" % timeit(lambda: ops.gattn_bwd(q, k, v, bk, bv, refs, i1, v1, bias, heads, hd,
                                                                    dout, gather=True, workspace=ws)))
    M = B * Q
    x = t(M, 256)
    w1 = t(512, 256)
    b1 = torch.zeros(512, device="cuda")
    print("fc1 GEMM+GELU(aux)   %.3f ms" % timeit(lambda: ops.linear_gelu_save(x, w1, b1)))
    print("fc1 GEMM identity    %.3f ms" % timeit(lambda: ops.linear(x, w1, b1)))
    keys, _ = ops.visible_coords(masks)
    sub = keys[:, ::6].contiguous()  # a sparse stage (~680 keys)
    print("knn refs->sparse     %.3f ms (%d keys)" % (timeit(lambda: ops.knn(refs, sub, 8)), sub.shape[1]))
    print("knn refs->stage0     %.3f ms (%d keys)" % (timeit(lambda: ops.knn(refs, keys, 8)), keys.shape[1]))


if __name__ == "__main__":
    main()
