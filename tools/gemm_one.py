"""One GEMM shape, for ncu: python tools/gemm_one.py M N K [fwd|gelu|bwd]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16249_b200 import ops  # noqa: E402
m, n, k = (int(a) for a in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "fwd"
x = torch.randn((m, k), device="cuda").to(torch.bfloat16)
w = (torch.randn((n, k), device="cuda") / k ** 0.5).to(torch.bfloat16)
b = torch.randn(n, device="cuda")
dy = torch.randn((m, n), device="cuda").to(torch.bfloat16)
for _ in range(3):
    if mode == "fwd":
        ops.linear(x, w, b)
    elif mode == "gelu":
        ops.linear_gelu_save(x, w, b)
    else:
        ops.linear_bwd(x, w, dy)
torch.cuda.synchronize()
