"""Quick device timing of the attention kernels (development probe, not the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import port
from paper_2602_16249_b200 import inputs, ops

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
grid, heads, hd = 256, 4, 32
coords = inputs.lattice_batch(B, grid)
N = coords.shape[1]
geom = ops.geometry(B, N, 16, 3)
P, CO, NB, RO, RC = [], [], [], [], []
for b in range(B):
    ci = port.cluster_index(coords[b], 16, 3)
    nb = ci["nbr_cl"]
    rev = [[] for _ in range(nb.shape[0])]
    for c in range(nb.shape[0]):
        for g in range(nb.shape[1]):
            rev[nb[c, g]].append(c)
    P.append(ci["members"]); CO.append(ci["cluster_of"]); NB.append(nb)
    RO.append(np.cumsum([0] + [len(r) for r in rev])); RC.append([c for r in rev for c in r])
dev = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.int32, device="cuda").contiguous()
index = ops.ClusterIndex(geom, dev(np.stack(P)), dev(np.stack(CO)), dev(np.stack(NB)),
                         dev(np.stack(RO)), dev(np.stack(RC)))
rng = np.random.default_rng(0)
q, k, v, do = (torch.randn(B, N, heads * hd, device="cuda").mul_(0.5).bfloat16() for _ in range(4))
bk, bv = (torch.randn(heads, hd, device="cuda").mul_(0.5).bfloat16() for _ in range(2))
bias = ops.BiasNet.from_numpy(inputs.bias_params(heads, 8, rng))
c = torch.as_tensor(coords, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
out, lse = ops.attn_fwd(geom, q, k, v, bk, bv, c, index.perm, index.nbr_cl, bias, heads, hd, workspace=ws)
grads = ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, heads, hd, out, lse, do, workspace=ws)
torch.cuda.synchronize()


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


D = heads * hd
fwd = timeit(lambda: ops.attn_fwd(geom, q, k, v, bk, bv, c, index.perm, index.nbr_cl, bias, heads,
                                  hd, out, lse, workspace=ws))
bwd = timeit(lambda: ops.attn_bwd(geom, q, k, v, bk, bv, c, index, bias, heads, hd, out, lse, do,
                                  grads, workspace=ws))
T = B * N
print(f"attn_fwd B={B} N={N} D={D}: {fwd*1e3:.1f} us  {T/fwd/1e6:.1f} Mtok/s  "
      f"{T*(8*D+4*heads+8)/fwd/1e6:.0f} GB/s alg")
print(f"attn_bwd: {bwd*1e3:.1f} us  {T/bwd/1e6:.1f} Mtok/s  {T*(16*D+8*heads+8)/bwd/1e6:.0f} GB/s alg")
