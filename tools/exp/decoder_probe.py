"""Decoder ops at the bench's side-measurement size (8 images x 65536 grid cells): one
interpolation fwd/bwd over 16384 encoder tokens and one decoder self attention fwd/bwd
(4 heads x 16, knn 8), for ncu captures of the §8(f) #2 kernels."""
import numpy as np
import torch

from paper_2602_16249_b200 import inputs, ops

dev = "cuda"
nb, g = 8, 256
cc = (np.arange(g) * 8.0 + 4.0).astype(np.float32)
q0 = np.stack(np.meshgrid(cc, cc), -1).reshape(1, -1, 2)
coords = torch.as_tensor(np.repeat(q0, nb, 0), device=dev).contiguous()
keys = torch.as_tensor(inputs.lattice_batch(nb, g, 0.75, 8, 1000), device=dev).contiguous()
N = coords.shape[1]
bf = torch.bfloat16
# interpolation (D = 128)
feats = torch.randn((nb, keys.shape[1], 128), device=dev).to(bf)
dout = torch.randn((nb, N, 128), device=dev).to(bf)
p = torch.tensor([1.0], device=dev)
iidx, ivalid = ops.knn(coords, keys, 8)
# decoder self attention
heads, hd = 4, 16
idx, valid = ops.knn(coords, coords, 8)
q, k, v, do = ((0.5 * torch.randn((nb, N, heads * hd), device=dev)).to(bf) for _ in range(4))
bk = torch.zeros((heads, hd), dtype=bf, device=dev)
bias = ops.BiasNet.from_numpy(inputs.bias_params(heads, 8, np.random.default_rng(1)), device=dev)
for _ in range(3):
    ops.interp_fwd(coords, keys, feats, iidx, ivalid, p)
    ops.interp_bwd(coords, keys, feats, iidx, ivalid, p, dout)
    ops.interp_bwd(coords, keys, feats, iidx, ivalid, p, dout, gather=True)
    ops.gattn_fwd(q, k, v, bk, bk, coords, idx, valid, bias, heads, hd)
    ops.gattn_bwd(q, k, v, bk, bk, coords, idx, valid, bias, heads, hd, do)
torch.cuda.synchronize()
print("ok")
