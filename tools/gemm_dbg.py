import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16249_b200 import ops
m, n, k = [int(a) for a in sys.argv[1:4]]
x = torch.randn((m, k), device="cuda").to(torch.bfloat16)
w = (torch.randn((n, k), device="cuda") / k ** 0.5).to(torch.bfloat16)
b = torch.randn(n, device="cuda")
y = ops.linear(x, w, b)
torch.cuda.synchronize()
ref = x.float() @ w.float().t() + b
print("rel", float((y.float() - ref).norm() / ref.norm()))
