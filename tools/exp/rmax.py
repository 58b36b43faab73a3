import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2602_16249_b200 import inputs, ops
coords = torch.as_tensor(inputs.lattice_batch(32, 256, 0.75, 8, seed0=1000), device='cuda')
B, N, _ = coords.shape
idx = ops.cluster_index(coords, 16, 3)
geom = ops.geometry(B, N, 16, 3)
pl = ops.attn_plan(geom, coords, idx, 4, 32, 8)
# rmax lives after qrec|items|count|blk in the plan buffer: recompute offsets like carve_plan
al = lambda x: (x + 255) & ~255
items = B * geom.n_clusters; qw = 32 + 2 * 48 + 8
off = al(items * qw * 4) + al(2 * items * 4) + al(8) + al(2 * ((items + 1023) // 1024) * 4)
print("rmax", pl.buf[off:off + 4].view(torch.int32).item())
q = pl.buf[:items * qw * 4].view(torch.int32).view(items, qw)
cls = q[:, 32 + 96 + 2].cpu().numpy()
print("classes", np.bincount(cls, minlength=3))
