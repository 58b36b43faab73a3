"""One tcgen05 linear launch per shape (for ncu captures of the §8(f) #1 kernel)."""
import sys

import torch

from paper_2602_16249_b200 import ops

m, n, k, act = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
x = torch.randn((m, k), device="cuda").to(torch.bfloat16)
w = torch.randn((n, k), device="cuda").to(torch.bfloat16)
for _ in range(3):
    ops.linear(x, w, act=act)
torch.cuda.synchronize()
