"""Times the training step's GEMM shapes through the C ABI (CUDA events, 20 reps after warm-up):
fwd, fwd+GELU-aux, dX + dW (split-K) + db, dW + db (profiles/r02k_gemm_ab.txt holds the A/B against
the CUTLASS builder GEMM this kernel replaced)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16249_b200 import ops  # noqa: E402

SHAPES = [(262144, 384, 128), (262144, 512, 128), (262144, 128, 512), (104832, 768, 256), (104832, 1024, 256),
          (104832, 256, 1024), (41920, 1536, 512), (41920, 2048, 512), (41920, 512, 2048), (16768, 4096, 1024),
          (16768, 1024, 4096), (786432, 256, 256), (524288, 512, 128)]


def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


out = []
for m, n, k in SHAPES:
    x = torch.randn((m, k), device="cuda").to(torch.bfloat16)
    w = (torch.randn((n, k), device="cuda") / k ** 0.5).to(torch.bfloat16)
    b = torch.randn(n, device="cuda")
    dy = torch.randn((m, n), device="cuda").to(torch.bfloat16)
    dw = torch.zeros((n, k), device="cuda")
    r = {"m": m, "n": n, "k": k}
    r["fwd"] = t(lambda: ops.linear(x, w, b))
    r["fwd_gelu"] = t(lambda: ops.linear_gelu_save(x, w, b))
    r["bwd"] = t(lambda: ops.linear_bwd(x, w, dy, dw=dw))
    r["bwd_w"] = t(lambda: ops.linear_bwd(x, w, dy, dw=dw, need_dx=False))
    fl = 2.0 * m * n * k
    r["fwd_tf"] = fl / r["fwd"] / 1e9
    r["bwd_tf"] = 2 * fl / r["bwd"] / 1e9
    out.append(r)
    print(json.dumps({kk: (round(v, 4) if isinstance(v, float) else v) for kk, v in r.items()}), flush=True)
    del x, w, dy, dw
