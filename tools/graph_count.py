import torch
from cuda.bindings import runtime as rt
g = torch.cuda.CUDAGraph()
x = torch.zeros(10, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    x.add_(1)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    x.add_(1)
    x.mul_(2)
raw = g.raw_cuda_graph()
print("raw", type(raw), raw)
h = rt.cudaGraph_t(init_value=raw)
r = rt.cudaGraphGetNodes(h, 0)
print("getnodes0", r)
r = rt.cudaGraphGetNodes(h, r[2])
print("getnodes", r)
for nd in r[1]:
    print(rt.cudaGraphNodeGetType(nd))
