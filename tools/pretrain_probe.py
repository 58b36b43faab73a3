"""AFFMAE-B pretraining step probe (BASELINE configs[2]): device-timed img/s of the whole
training step (masks, encode, decode, deep supervision, loss, backward, AdamW) through the
torch-free model API, eager and as a CUDA graph.

    python tools/pretrain_probe.py --batch 16 --steps 10 [--image 1024] [--no-graph]
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_16249_b200 import capi, devmem  # noqa: E402
from paper_2602_16249_b200.model import Model, affmae_b, step_mask_seed  # noqa: E402


def synth_into(m, B, size, seed0, stream):
    L = capi.lib()
    L.affmae_synth_images_workspace.restype = C.c_size_t
    ws_bytes = L.affmae_synth_images_workspace(C.c_int64(B), C.c_int64(size))
    ws = devmem.DeviceBuffer(ws_bytes)
    seeds = np.arange(seed0, seed0 + B, dtype=np.uint64)
    capi.check(L.affmae_synth_images(seeds.ctypes.data_as(C.c_void_p), C.c_int64(B), C.c_int64(size),
                                     C.c_void_p(m.images_ptr), C.c_void_p(ws.ptr), C.c_size_t(ws_bytes),
                                     C.c_void_p(stream)), "synth_images")
    devmem.sync(stream)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--image", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    cfg = affmae_b(image=a.image, batch=a.batch, total_steps=1000)
    t0 = time.time()
    m = Model(cfg)
    print(f"create {time.time() - t0:.1f}s  params {m.n_values}  tokens {m.tokens}  masked {m.masked}  "
          f"device {m.device_bytes / 2**30:.2f} GiB", flush=True)
    st = devmem.stream_create()
    synth_into(m, a.batch, a.image, 400, st)
    step = 0

    def one(graph):
        nonlocal step
        seeds = [step_mask_seed(1, step * a.batch + i) for i in range(a.batch)]
        m.make_masks(seeds, stream=st)
        m.train_step(use_graph=graph, stream=st, read_loss=False)
        step += 1

    for mode in (["eager"] if a.no_graph else ["eager", "graph"]):
        g = mode == "graph"
        for _ in range(a.warmup):
            one(g)
        devmem.sync(st)
        e0, e1 = devmem.Event(), devmem.Event()
        e0.record(st)
        for _ in range(a.steps):
            one(g)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_ms(e1) / a.steps
        loss = devmem.d2h(m._loss_buf().ptr, (3,), np.float32, st)
        print(f"{mode}: {ms:.2f} ms/step  {a.batch / ms * 1e3:.1f} img/s  loss {loss}", flush=True)


if __name__ == "__main__":
    main()
