import torch, time
n_in, n_out = 650_544_160, 788_955_136
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory(); ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device='cuda'); do = torch.empty(n_out, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(both=True, h2d=True, d2h=True):
    torch.cuda.synchronize(); t=time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize(); return time.perf_counter()-t
for _ in range(2): run()
print("h2d only GB/s", n_in/run(d2h=False)/1e9, "d2h only GB/s", n_out/run(h2d=False)/1e9, "both ms", run()*1e3)
