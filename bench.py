#!/usr/bin/env python3
"""Benchmark of the AFFMAE hot path on B200 (driver contract: one JSON line).

Workload = BASELINE.json configs[1], the standalone cluster-attention + KNN-merge
op sweep, at its headline point: per GPU B images of a 256x256 patch grid with a
75% Perlin mask (N = 16384 visible tokens per image, exact mask counts), D = 128
(4 heads x 32), K = 48 neighbours (cluster 16 x groups 3), BiasNet hidden 8,
merge d_s = 0.4, k_m = 8.  One step = the whole hot path over the batch:
    cluster index build -> cluster attention fwd -> attention bwd ->
    select_retained -> merge_plan -> merge pool fwd -> merge pool bwd
(synthetic inputs; q/k/v/blanks ~ 0.5 N(0,1) bf16, dO ~ N(0,1), scores ~ U(0.1, 0.9);
merge features = the attention output).  Inputs per step (q, k, v, dO: 4 x B x N x D
bf16 = 537 MB at B = 32) exceed the 126 MB L2, so no flush is needed.

value  device-resident tokens/s (all ranks' tokens / max-over-ranks device time)
e2e    the same through the C ABI with HOST buffers: pinned H2D of every input and
       D2H of every output inside the timed region.
--impl reference  times the reference's own CPU implementation (oracle/_ref, the
       unmodified reference C++ compiled by oracle/Makefile) on all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "cluster-attn tokens/s fwd+bwd"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=32, help="images per GPU")
    ap.add_argument("--grid", type=int, default=256, help="patch grid side (75%% masked)")
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--head-dim", type=int, default=32)
    ap.add_argument("--cluster", type=int, default=16)
    ap.add_argument("--groups", type=int, default=3)
    ap.add_argument("--hidden", type=int, default=8)
    ap.add_argument("--d-s", type=float, default=0.4)
    ap.add_argument("--k-m", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=8, help="image chunks pipelined H2D|compute|D2H")
    ap.add_argument("--e2e-ramp", type=str, default="",
                    help="image counts of the first chunks (and, reversed, the last ones): small chunks "
                         "at both ends shorten the pipeline fill and drain")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--streams", type=int, default=1,
                    help="independent image groups per GPU, each on its own stream pair (images never "
                         "interact, so the groups' latency-bound phases overlap each other)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--interp-images", type=int, default=8,
                    help="images of the side measurement of the interpolation op (SURVEY §8(f) #2); 0 = off")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="CPU baseline sample budget")
    ap.add_argument("--pretrain-batch", type=int, default=64, help="AFFMAE-B 1024^2 images per step (0: skip)")
    ap.add_argument("--pretrain-steps", type=int, default=5)
    ap.add_argument("--tiny-batch", type=int, default=64, help="AFF-tiny 224^2 images per step (0: skip)")
    ap.add_argument("--no-parity", action="store_true", help="skip the same-run oracle check")
    return ap.parse_args()


def workload_config(a, world):
    return {"workload": "configs[1] op sweep point: cluster index + cluster attention fwd+bwd "
                        "+ KNN merge (select, plan, pool fwd+bwd)",
            "images_per_gpu": a.batch, "global_images": a.batch * world,
            "grid": a.grid, "mask_ratio": 0.75, "tokens_per_image": None,
            "dim": a.heads * a.head_dim, "heads": a.heads, "head_dim": a.head_dim,
            "neighbours": a.cluster * a.groups, "cluster": a.cluster, "groups": a.groups,
            "bias_hidden": a.hidden, "d_s": a.d_s, "k_m": a.k_m,
            "l2": "inputs per step > 126 MB L2 (no flush needed)",
            "parallelism": f"dp{world} (images sharded, no data-path collective)",
            "image_streams": getattr(a, "streams", 1)}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled from a
    thread every 5 ms (the timed region of a default run is tens of ms), nvidia-smi as the
    fallback."""

    REASONS = {  # NVML clocks-event-reason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self._stop = threading.Event()
        self._thr = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception:
            self._nvml = None

    def _poll_nvml(self):
        nv = self._nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                try:
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except AttributeError:
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                rs = {n for b, n in self.REASONS.items() if bits & b}
                self.samples.append((float(sm), float(mx), rs))
            except Exception:
                pass
            self._stop.wait(0.005)

    def _poll_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout
                parts = [x.strip() for x in out.strip().split(",")]
                if len(parts) >= 6 and parts[0].replace(".", "").isdigit():
                    rs = {names[i - 2] for i in range(2, 6) if parts[i].lower() == "active"}
                    self.samples.append((float(parts[0]), float(parts[1]), rs))
            except Exception:
                pass
            self._stop.wait(0.05)

    def start(self):
        self._thr = threading.Thread(target=self._poll_nvml if self._nvml else self._poll_smi, daemon=True)
        self._thr.start()

    def stop(self):
        self._stop.set()
        if self._thr is not None:
            self._thr.join(timeout=10)

    def summary(self):
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples]
        reasons = sorted(set().union(*[x[2] for x in self.samples])) if self.samples else []
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi",
                "window": "timed region + 0.25 s of the same step" if getattr(self, "extended", False)
                          else "timed region"}


# --------------------------------------------------------------- workload
def make_inputs(a, rank):
    from paper_2602_16249_b200 import inputs
    rng = np.random.default_rng(1234 + rank)
    from paper_2602_16249_b200 import dist as pdist
    # global image index -> mask seed, so results do not depend on the rank count
    coords = inputs.lattice_batch(a.batch, a.grid, 0.75, 8,
                                  seed0=pdist.mask_seed(pdist.image_range(a.batch, rank, max(rank + 1, 1))[0]))
    B, N, _ = coords.shape
    hd = a.heads * a.head_dim
    host = dict(
        coords=coords,
        q=(0.5 * rng.standard_normal((B, N, hd))).astype(np.float32),
        k=(0.5 * rng.standard_normal((B, N, hd))).astype(np.float32),
        v=(0.5 * rng.standard_normal((B, N, hd))).astype(np.float32),
        dout=rng.standard_normal((B, N, hd)).astype(np.float32),
        bk=(0.5 * rng.standard_normal((a.heads, a.head_dim))).astype(np.float32),
        bv=(0.5 * rng.standard_normal((a.heads, a.head_dim))).astype(np.float32),
        scores=rng.uniform(0.1, 0.9, (B, N)).astype(np.float32),
        bias=inputs.bias_params(a.heads, a.hidden, rng),
    )
    return host


def algorithmic_bytes(a, N):
    """Per-token algorithmic HBM bytes, SURVEY.md §8(d)'s figures."""
    D, h = a.heads * a.head_dim, a.heads
    return {
        "attn_fwd": 8 * D + 4 * h + 8,         # q,k,v read + o write (bf16), lse write, coords
        # §8(d): 16 D + 4h -- q,k,v,o,dO read + dq,dk,dv write (bf16) + lse; this backward does
        # not read o (D = rowsum(P dP) is recomputed), so it moves 14 D + 4h + 8 of them
        "attn_bwd": 16 * D + 4 * h,
        "index": 8 + 4 + 4 + 4 * a.groups / a.cluster,  # coords in; perm, cluster_of, nbr ids out
        "merge": 4 + 8 + 2 * D + 4 + a.d_s * (4 + 4 * D + 12 * a.k_m),  # fwd side
    }


# ------------------------------------------------------------------ ours
def run_ours(a, rank, world, dist):
    import torch
    from paper_2602_16249_b200 import dist as pdist
    from paper_2602_16249_b200 import ops
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    host = make_inputs(a, rank)
    B, N, _ = host["coords"].shape
    bf = torch.bfloat16

    def to_dev(x, dt):
        return torch.as_tensor(x, dtype=dt, device=dev).contiguous()

    coords = to_dev(host["coords"], torch.float32)
    q, k, v, dout = (to_dev(host[n], bf) for n in ("q", "k", "v", "dout"))
    bk, bv = to_dev(host["bk"], bf), to_dev(host["bv"], bf)
    scores = to_dev(host["scores"], torch.float32)
    bias = ops.BiasNet.from_numpy(host["bias"], device=dev)
    p_merge = torch.tensor([1.0], dtype=torch.float32, device=dev)
    h, d = a.heads, a.head_dim
    geom = ops.geometry(B, N, a.cluster, a.groups)
    R = ops.retained_count(N, a.d_s)
    dpooled = torch.randn((B, R, 2 * h * d), device=dev).to(bf)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out_buf = torch.empty_like(q)
    lse_buf = torch.empty((B, N, h), dtype=torch.float32, device=dev)
    grads = ops.AttnGrads.zeros_like(q, bk, bias)
    plan_buf = torch.empty(64 << 20, dtype=torch.uint8, device=dev)

    phases = ["index", "attn_fwd", "attn_bwd", "merge"]

    def step(ev=None):
        if ev:
            ev[0].record()
        idx = ops.cluster_index(coords, a.cluster, a.groups, workspace=ws)
        if ev:
            ev[1].record()
        plan = ops.attn_plan(geom, coords, idx, h, d, a.hidden, buf=plan_buf)
        out, lse = ops.attn_fwd(geom, q, k, v, bk, bv, coords, idx.perm, idx.nbr_cl, bias, h, d,
                                out=out_buf, lse=lse_buf, workspace=ws, plan=plan)
        if ev:
            ev[2].record()
        ops.attn_bwd(geom, q, k, v, bk, bv, coords, idx, bias, h, d, out, lse, dout, grads=grads,
                     workspace=ws, plan=plan)
        if ev:
            ev[3].record()
        ret = ops.select_retained(scores, a.d_s)
        plan = ops.merge_plan(coords, ret, a.k_m)
        pooled = ops.merge_pool_fwd(out, scores, p_merge, plan)
        dfe, dsc, dp = ops.merge_pool_bwd(out, scores, p_merge, plan, dpooled)
        if ev:
            ev[4].record()
        return out, lse, grads, pooled, dfe, dsc, dp

    side = torch.cuda.Stream(device=dev)

    def step_dag():
        """The same step as a two-stream DAG: selection + merge plan depend only on scores
        and coordinates, the pool fwd/bwd only on the attention output, so they run beside the
        index build and the attention backward."""
        cur = torch.cuda.current_stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            ret = ops.select_retained(scores, a.d_s)
            mplan = ops.merge_plan(coords, ret, a.k_m)
        idx = ops.cluster_index(coords, a.cluster, a.groups, workspace=ws)
        plan = ops.attn_plan(geom, coords, idx, h, d, a.hidden, buf=plan_buf)
        out, lse = ops.attn_fwd(geom, q, k, v, bk, bv, coords, idx.perm, idx.nbr_cl, bias, h, d,
                                out=out_buf, lse=lse_buf, workspace=ws, plan=plan)
        fwd_done = torch.cuda.Event()
        fwd_done.record(cur)
        with torch.cuda.stream(side):
            side.wait_event(fwd_done)
            pooled = ops.merge_pool_fwd(out, scores, p_merge, mplan)
            dfe, dsc, dp = ops.merge_pool_bwd(out, scores, p_merge, mplan, dpooled)
        ops.attn_bwd(geom, q, k, v, bk, bv, coords, idx, bias, h, d, out, lse, dout, grads=grads,
                     workspace=ws, plan=plan)
        cur.wait_stream(side)
        return out, lse, grads, pooled, dfe, dsc, dp

    # --streams S: the batch as S independent image groups, each the same DAG on its own
    # stream pair, sharing nothing but the (read-only) inputs; every group writes its own slice
    # of the outputs and its own parameter-gradient partials, summed at the end of the step
    S = max(1, min(a.streams, B))
    gb = [(B * g // S, B * (g + 1) // S) for g in range(S)]
    groups = []
    if S > 1:
        for (b0, b1) in gb:
            gq = dict(geom=ops.geometry(b1 - b0, N, a.cluster, a.groups),
                      ws=torch.empty(256 << 20, dtype=torch.uint8, device=dev),
                      plan_buf=torch.empty(64 << 20, dtype=torch.uint8, device=dev),
                      main=torch.cuda.Stream(device=dev), side=torch.cuda.Stream(device=dev),
                      grads=ops.AttnGrads(grads.dq[b0:b1], grads.dk[b0:b1], grads.dv[b0:b1],
                                          *[torch.zeros_like(t) for t in (grads.dblank_k, grads.dblank_v,
                                                                          grads.dw1, grads.db1, grads.dw2,
                                                                          grads.db2, grads.dblank)]),
                      pooled=None)
            groups.append(gq)

    def group_dag(g):
        b0, b1 = gb[g]
        st = groups[g]
        cur, side_g = st["main"], st["side"]
        sl = slice(b0, b1)
        side_g.wait_stream(cur)
        with torch.cuda.stream(side_g):
            ret = ops.select_retained(scores[sl], a.d_s)
            mplan = ops.merge_plan(coords[sl], ret, a.k_m)
        idx = ops.cluster_index(coords[sl], a.cluster, a.groups, workspace=st["ws"])
        plan = ops.attn_plan(st["geom"], coords[sl], idx, h, d, a.hidden, buf=st["plan_buf"])
        out, lse = ops.attn_fwd(st["geom"], q[sl], k[sl], v[sl], bk, bv, coords[sl], idx.perm, idx.nbr_cl, bias,
                                h, d, out=out_buf[sl], lse=lse_buf[sl], workspace=st["ws"], plan=plan)
        fwd_done = torch.cuda.Event()
        fwd_done.record(cur)
        with torch.cuda.stream(side_g):
            side_g.wait_event(fwd_done)
            pooled = ops.merge_pool_fwd(out, scores[sl], p_merge, mplan)
            dfe, dsc, dp = ops.merge_pool_bwd(out, scores[sl], p_merge, mplan, dpooled[sl])
        ops.attn_bwd(st["geom"], q[sl], k[sl], v[sl], bk, bv, coords[sl], idx, bias, h, d, out, lse, dout[sl],
                     grads=st["grads"], workspace=st["ws"], plan=plan)
        cur.wait_stream(side_g)
        return pooled, dfe, dsc, dp

    def step_groups():
        cur = torch.cuda.current_stream(dev)
        res = []
        for g in range(S):
            groups[g]["main"].wait_stream(cur)
            with torch.cuda.stream(groups[g]["main"]):
                res.append(group_dag(g))
        for g in range(S):
            cur.wait_stream(groups[g]["main"])
        # parameter-gradient partials of the groups -> the step's gradients
        for name in ("dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank"):
            tot = getattr(grads, name)
            tot.copy_(getattr(groups[0]["grads"], name))
            for g in range(1, S):
                tot.add_(getattr(groups[g]["grads"], name))
        return res

    if S > 1:
        step_dag_single = step_dag
        step_dag = step_groups  # noqa: F811 (the timed and captured step)

    # warm-up (also primes the caching allocator) + per-phase timing pass (sequential)
    for _ in range(max(1, a.warmup)):
        step()
        step_dag()
    torch.cuda.synchronize()
    n_ph = 5
    phase_ms = {p: [] for p in phases}
    for _ in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_ph)]
        step(ev)
        torch.cuda.synchronize()
        for i, p in enumerate(phases):
            phase_ms[p].append(ev[i].elapsed_time(ev[i + 1]))

    # CUDA graph of one step (launch-bound small kernels), eager fallback
    graph = None
    launches = None
    if not a.no_graph:
        try:
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step_dag()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            try:
                graph = torch.cuda.CUDAGraph(keep_graph=True)
            except TypeError:  # older torch
                graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step_dag()
            torch.cuda.synchronize()
            launches = count_graph_kernels(graph)
            if hasattr(graph, "instantiate"):
                try:
                    graph.instantiate()
                except RuntimeError:
                    pass
        except Exception as e:  # pragma: no cover - capture is best effort
            print(f"[bench] CUDA graph capture failed ({e}); eager launches", file=sys.stderr)
            graph = None

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step_dag()

    for _ in range(a.warmup):
        run_step()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    e0.record()
    for _ in range(a.steps):
        run_step()
    e1.record()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = e0.elapsed_time(e1) / a.steps
    clocks.stop()
    if len(clocks.samples) < 3:
        # timed region shorter than the sampler can resolve: keep the same step running
        # (untimed) for ~0.25 s under the sampler so the clock record reflects this load
        ext = ClockSampler(dev.index)
        ext.start()
        t_end = time.perf_counter() + 0.25
        while time.perf_counter() < t_end:
            for _ in range(10):
                run_step()
            torch.cuda.synchronize()
        ext.stop()
        clocks.samples += ext.samples
        clocks.extended = True
    ms_max = pdist.max_over_ranks(ms, dist, dev)
    tokens_all = B * N * world
    value = tokens_all / (ms_max * 1e-3)

    # e2e through the C ABI with host buffers (pinned H2D + D2H inside the timed region)
    e2e = run_e2e(a, host, dev, geom, h, d, ws, world, dist) if a.e2e_steps > 0 else {}
    interp = run_interp(a, host, dev) if a.interp_images > 0 else None
    adamw = run_adamw(dev) if a.interp_images > 0 else None
    linear = run_linear(dev) if a.interp_images > 0 else None
    gattn = run_gattn(a, host, dev) if a.interp_images > 0 else None
    masks = run_masks(a, dev) if a.interp_images > 0 else None

    res = dict(value=value, ms=ms_max, phase_ms={p: float(np.median(v)) for p, v in phase_ms.items()},
               clocks=clocks.summary(), e2e=e2e, N=N, B=B, launches=launches,
               graph=graph is not None, interp=interp, adamw=adamw, linear=linear, gattn=gattn, masks=masks)
    return res


def count_graph_kernels(graph):
    """Kernel nodes in the captured step (our launches; the step holds no torch compute)."""
    try:
        from cuda.bindings import runtime as rt
    except ImportError:  # pragma: no cover
        try:
            from cuda import cudart as rt
        except ImportError:
            return None
    try:
        g = rt.cudaGraph_t(init_value=graph.raw_cuda_graph())
        err, nodes, n = rt.cudaGraphGetNodes(g, 0)
        err, nodes, n = rt.cudaGraphGetNodes(g, n)
        kern = 0
        for nd in nodes:
            err, ty = rt.cudaGraphNodeGetType(nd)
            if ty == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
                kern += 1
        return kern
    except Exception:
        return None


def run_interp(a, host, dev, k=8, reps=10):
    """Side measurement (not part of the step): the decoder's softmax interpolation
    (make_interp_op) of the encoder tokens onto every patch centre of the grid, knn rows
    built once; fwd and bwd (scattered reductions, and the reverse-CSR gather variant with
    its per-call CSR build) timed with CUDA events over `reps` calls each."""
    import torch
    from paper_2602_16249_b200 import capi, ops
    nb = min(a.interp_images, host["coords"].shape[0])
    keys = torch.as_tensor(host["coords"][:nb], device=dev).contiguous()
    g = a.grid
    cc = (np.arange(g) * 8.0 + 4.0).astype(np.float32)
    q = np.stack(np.meshgrid(cc, cc), -1).reshape(1, -1, 2)
    queries = torch.as_tensor(np.repeat(q, nb, 0), device=dev).contiguous()
    D = a.heads * a.head_dim
    feats = torch.randn((nb, keys.shape[1], D), device=dev).to(torch.bfloat16)
    dout = torch.randn((nb, queries.shape[1], D), device=dev).to(torch.bfloat16)
    p = torch.tensor([1.0], dtype=torch.float32, device=dev)
    idx, valid = ops.knn(queries, keys, k)
    dfe = torch.zeros((nb, keys.shape[1], D), dtype=torch.float32, device=dev)
    dp = torch.zeros(1, dtype=torch.float32, device=dev)
    dq = torch.zeros((nb, queries.shape[1], 2), dtype=torch.float32, device=dev)
    for _ in range(2):
        ops.interp_fwd(queries, keys, feats, idx, valid, p)
        ops.interp_bwd(queries, keys, feats, idx, valid, p, dout, dfeats=dfe, dp=dp, dqueries=dq, gather=False)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(reps):
        ops.interp_fwd(queries, keys, feats, idx, valid, p)
    ev[1].record()
    for _ in range(reps):
        ops.interp_bwd(queries, keys, feats, idx, valid, p, dout, dfeats=dfe, dp=dp, dqueries=dq, gather=False)
    ev[2].record()
    for _ in range(2):
        ops.interp_bwd(queries, keys, feats, idx, valid, p, dout, dfeats=dfe, dp=dp, dqueries=dq, gather=True)
    nbytes = capi.lib().affmae_interp_bwd_gather_workspace(nb, queries.shape[1], keys.shape[1], k)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ev3 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev3[0].record()
    for _ in range(reps):
        ops.interp_bwd(queries, keys, feats, idx, valid, p, dout, dfeats=dfe, dp=dp, dqueries=dq, gather=True,
                       workspace=ws)
    ev3[1].record()
    torch.cuda.synchronize()
    fwd_ms, bwd_ms = ev[0].elapsed_time(ev[1]) / reps, ev[1].elapsed_time(ev[2]) / reps
    bwd_gather_ms = ev3[0].elapsed_time(ev3[1]) / reps
    nq = nb * queries.shape[1]
    # algorithmic bytes per query: query xy 8 + k (idx 4 + valid 1) + output row 2D (fwd);
    # + cotangent row 2D and dq 8 (bwd); each key row read once and (bwd) written once in fp32
    kb = nb * keys.shape[1]
    fwd_bytes = nq * (8 + 5 * k + 2 * D) + kb * (8 + 2 * D)
    bwd_bytes = nq * (8 + 5 * k + 2 * D + 8) + kb * (8 + 2 * D + 2 * 4 * D)
    return {"images": nb, "queries_per_image": int(queries.shape[1]), "keys_per_image": int(keys.shape[1]),
            "k": k, "dim": D, "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "bwd_gather_ms": bwd_gather_ms,
            "fwd_queries_per_s": nq / (fwd_ms * 1e-3), "bwd_queries_per_s": nq / (bwd_ms * 1e-3),
            "fwd_gbs": fwd_bytes / (fwd_ms * 1e-3) / 1e9, "bwd_gbs": bwd_bytes / (bwd_ms * 1e-3) / 1e9,
            "bwd_gather_gbs": bwd_bytes / (bwd_gather_ms * 1e-3) / 1e9,
            "note": "side measurement of SURVEY §8(f) #2, not part of the step or its value"}


def run_gattn(a, host, dev, k=8, heads=4, head_dim=16, hidden=8, reps=10):
    """Side measurement: the decoder's self attention over knn rows
    (pipeline.cpp:493, 522-525; DecoderConfig defaults dim 64 = 4 heads x 16, self_k 8) on
    every patch centre of `interp_images` images; fwd and bwd timed with CUDA events."""
    import torch
    from paper_2602_16249_b200 import inputs, ops
    nb = min(a.interp_images, host["coords"].shape[0])
    g = a.grid
    cc = (np.arange(g) * 8.0 + 4.0).astype(np.float32)
    q0 = np.stack(np.meshgrid(cc, cc), -1).reshape(1, -1, 2)
    coords = torch.as_tensor(np.repeat(q0, nb, 0), device=dev).contiguous()
    N, D = coords.shape[1], heads * head_dim
    idx, valid = ops.knn(coords, coords, k)
    bf = torch.bfloat16
    q, kk, v, do = (0.5 * torch.randn((nb, N, D), device=dev)).to(bf), (0.5 * torch.randn((nb, N, D), device=dev)).to(bf), \
        (0.5 * torch.randn((nb, N, D), device=dev)).to(bf), torch.randn((nb, N, D), device=dev).to(bf)
    bk, bv = torch.zeros((heads, head_dim), dtype=bf, device=dev), torch.zeros((heads, head_dim), dtype=bf, device=dev)
    rng = np.random.default_rng(7)
    bias = ops.BiasNet.from_numpy(inputs.bias_params(heads, hidden, rng), device=dev)
    grads = ops.gattn_bwd(q, kk, v, bk, bv, coords, idx, valid, bias, heads, head_dim, do)
    for _ in range(2):
        ops.gattn_fwd(q, kk, v, bk, bv, coords, idx, valid, bias, heads, head_dim)
        ops.gattn_bwd(q, kk, v, bk, bv, coords, idx, valid, bias, heads, head_dim, do, grads=grads)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(reps):
        ops.gattn_fwd(q, kk, v, bk, bv, coords, idx, valid, bias, heads, head_dim)
    ev[1].record()
    for _ in range(reps):
        ops.gattn_bwd(q, kk, v, bk, bv, coords, idx, valid, bias, heads, head_dim, do, grads=grads)
    ev[2].record()
    torch.cuda.synchronize()
    fwd_ms, bwd_ms = ev[0].elapsed_time(ev[1]) / reps, ev[1].elapsed_time(ev[2]) / reps
    nt = nb * N
    # algorithmic bytes per token: q / k / v rows 2D each, xy 8, rows k*(4+1), out 2D + lse 4h (fwd);
    # + dout 2D, dq 2D, dk / dv fp32 read-modify-write 16D (bwd)
    fwd_bytes = nt * (8 * D + 8 + 5 * k + 4 * heads)
    bwd_bytes = nt * (10 * D + 8 + 5 * k + 16 * D)
    return {"images": nb, "tokens_per_image": N, "k": k, "heads": heads, "head_dim": head_dim,
            "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "fwd_tokens_per_s": nt / (fwd_ms * 1e-3),
            "bwd_tokens_per_s": nt / (bwd_ms * 1e-3), "fwd_gbs": fwd_bytes / (fwd_ms * 1e-3) / 1e9,
            "bwd_gbs": bwd_bytes / (bwd_ms * 1e-3) / 1e9,
            "note": "side measurement of SURVEY §8(f) #2, not part of the step or its value"}


def run_masks(a, dev, reps=10):
    """Side measurement: the step's Perlin masks and stage-0 coordinates built
    on the device for all `batch` images (host gradient table + field + exact-count select +
    lattice compaction), against the host numpy restatement's time for the same masks."""
    import torch
    from paper_2602_16249_b200 import inputs, ops
    seeds = [1000 + b for b in range(a.batch)]
    for _ in range(2):
        m = ops.perlin_masks(seeds, a.grid, 0.75, device=dev)
        ops.visible_coords(m, nvis=a.grid * a.grid - int(round(0.75 * a.grid * a.grid)))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        m = ops.perlin_masks(seeds, a.grid, 0.75, device=dev)
        ops.visible_coords(m, nvis=a.grid * a.grid - int(round(0.75 * a.grid * a.grid)))
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    t0 = time.perf_counter()
    inputs.lattice_batch(4, a.grid, 0.75, 8, seed0=1000)
    host_ms = (time.perf_counter() - t0) * 1e3 * a.batch / 4
    return {"images": a.batch, "grid": a.grid, "ms": ms, "host_numpy_ms": host_ms,
            "note": "side measurement of SURVEY §8(f) #4 (includes the per-call workspace allocation), not part of the step"}


def run_linear(dev, reps=20):
    """Side measurement: the tcgen05 linear layer at the op sweep's MLP shape
    (all 32 x 16384 tokens, D = 128 -> 4D with bias + GELU fused; HBM-bound at ~100 flop/B) and
    at a compute-bound 8192^3, against the measured bf16 tensor peak."""
    import torch
    from paper_2602_16249_b200 import ops
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        peaks = {}
    tc_peak = float(peaks.get("bf16_tflops") or 1644.8)
    hbm_peak = float(peaks.get("hbm_gbs") or 6553.6)
    out = {}
    for name, (m, n, k, act) in {"mlp_fc1": (32 * 16384, 512, 128, "gelu"),
                                 "square_8192": (8192, 8192, 8192, "none")}.items():
        x = torch.randn((m, k), device=dev).to(torch.bfloat16)
        w = (torch.randn((n, k), device=dev) / k ** 0.5).to(torch.bfloat16)
        b = torch.zeros(n, dtype=torch.float32, device=dev)
        for _ in range(2):
            ops.linear(x, w, b, act=act)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ops.linear(x, w, b, act=act)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
        gbs = 2.0 * (m * k + n * k + m * n) / (ms * 1e-3) / 1e9
        out[name] = {"m": m, "n": n, "k": k, "act": act, "ms": ms, "tflops": tf, "tc_frac": tf / tc_peak,
                     "gbs": gbs, "hbm_frac": gbs / hbm_peak}
        del x, w, b
    out["note"] = "side measurement of SURVEY §8(f) #1 (tcgen05 linear + fused bias/GELU), not part of the step"
    return out


def run_adamw(dev, params=91_000_000, reps=20):
    """Side measurement: one fused AdamW step over an AFF-B-sized parameter set
    (~91 M fp32, matrices and vectors), 28 algorithmic bytes per parameter, against the HBM peak."""
    import torch
    from paper_2602_16249_b200 import ops
    shapes = []
    left = params
    while left > 0:  # 1024x1024 matrices plus one bias vector each, like the dense layers
        n = min(left, 1024 * 1024)
        shapes.append((max(2, n // 1024), 1024) if n >= 2048 else (n,))
        left -= int(np.prod(shapes[-1]))
        if left > 0:
            shapes.append((1024,))
            left -= 1024
    opt = ops.AdamW(shapes, total_steps=1000, device=dev)
    opt.grad.normal_()
    opt.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        opt.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    n = sum(int(np.prod(s)) for s in shapes)
    gbs = 28.0 * n / (ms * 1e-3) / 1e9
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 6553.6
    return {"params": n, "tensors": len(shapes), "ms": ms, "gbs": gbs, "hbm_frac": gbs / float(peak),
            "note": "side measurement of SURVEY §8(f) #3 (fused AdamW), not part of the step"}


def e2e_bounds(B, chunks, ramp):
    """Image ranges of the e2e chunks: `ramp` sizes first, the same reversed last, and the rest
    split into `chunks` near-equal chunks (the D2H stream can start after one small chunk and
    the last results leave right after the last small chunk's compute)."""
    rs = [int(x) for x in str(ramp).split(",") if x.strip()] if ramp else []
    if sum(rs) * 2 >= B:
        rs = []
    sizes = list(rs)
    mid = B - 2 * sum(rs)
    nmid = max(1, min(chunks, mid))
    sizes += [mid * (c + 1) // nmid - mid * c // nmid for c in range(nmid)]
    sizes += rs[::-1]
    bounds, b0 = [], 0
    for sz in sizes:
        if sz > 0:
            bounds.append((b0, b0 + sz))
            b0 += sz
    return bounds


def run_e2e(a, host, dev, geom, h, d, ws, world, dist):
    """The same step through the C ABI from HOST buffers: every input H2D and every output D2H
    inside the timed region.  Images are independent, so the batch is processed in chunks on
    three streams -- H2D of chunk c+1 | compute of chunk c | D2H of chunk c-1 -- and the PCIe
    copies in both directions overlap each other and the kernels."""
    import torch
    from paper_2602_16249_b200 import dist as pdist
    from paper_2602_16249_b200 import ops
    bf = torch.bfloat16
    pin = {}
    for n in ("q", "k", "v", "dout"):
        pin[n] = torch.from_numpy(host[n]).to(bf).pin_memory()
    pin["coords"] = torch.from_numpy(host["coords"]).pin_memory()
    pin["scores"] = torch.from_numpy(host["scores"]).pin_memory()
    B, N = pin["scores"].shape
    R = ops.retained_count(N, a.d_s)
    pin["dpooled"] = torch.randn((B, R, 2 * h * d)).to(bf).pin_memory()
    small = {n: torch.from_numpy(host[n]).to(bf).pin_memory() for n in ("bk", "bv")}
    hb = {n: torch.from_numpy(np.ascontiguousarray(host["bias"][n])).pin_memory()
          for n in ("w1", "b1", "w2", "b2", "blank")}
    hd_ = h * d
    outs_h = dict(out=torch.empty((B, N, hd_), dtype=bf).pin_memory(),
                  lse=torch.empty((B, N, h), dtype=torch.float32).pin_memory(),
                  dq=torch.empty((B, N, hd_), dtype=bf).pin_memory(),
                  dk=torch.empty((B, N, hd_), dtype=bf).pin_memory(),
                  dv=torch.empty((B, N, hd_), dtype=bf).pin_memory(),
                  pooled=torch.empty((B, R, 2 * hd_), dtype=bf).pin_memory(),
                  dfeats=torch.empty((B, N, hd_), dtype=bf).pin_memory(),
                  dscores=torch.empty((B, N), dtype=torch.float32).pin_memory())
    h2d = sum(t.numel() * t.element_size() for t in list(pin.values()) + list(small.values())
              + list(hb.values()))
    d2h = sum(t.numel() * t.element_size() for t in outs_h.values())

    bounds = e2e_bounds(B, a.e2e_chunks, a.e2e_ramp)
    nch = len(bounds)
    cgeom = {}
    for (b0, b1) in bounds:
        if b1 - b0 not in cgeom:
            cgeom[b1 - b0] = ops.geometry(b1 - b0, N, a.cluster, a.groups)
    s_in, s_cmp, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
    # device buffers per chunk (no reuse hazards between the streams)
    dbuf = [{n: torch.empty((b1 - b0,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
             for n, t in pin.items()} for (b0, b1) in bounds]
    dsmall = {n: torch.empty_like(t, device=dev) for n, t in small.items()}
    dhb = {n: torch.empty_like(t, device=dev) for n, t in hb.items()}
    p_merge = torch.ones(1, dtype=torch.float32, device=dev)
    plan_buf = torch.empty(64 << 20, dtype=torch.uint8, device=dev)

    bias = ops.BiasNet(**dhb)
    outs_d = [None] * nch

    s_side = torch.cuda.Stream(device=dev)

    def chunk_compute(c):
        """The op chain of one chunk (device buffers in, device results out), as the same
        two-stream DAG as the device-resident step."""
        b0, b1 = bounds[c]
        dv_ = dbuf[c]
        g = cgeom[b1 - b0]
        cur = torch.cuda.current_stream(dev)
        s_side.wait_stream(cur)
        with torch.cuda.stream(s_side):
            ret = ops.select_retained(dv_["scores"], a.d_s)
            mplan = ops.merge_plan(dv_["coords"], ret, a.k_m)
        idx = ops.cluster_index(dv_["coords"], a.cluster, a.groups, workspace=ws)
        plan = ops.attn_plan(g, dv_["coords"], idx, h, d, a.hidden, buf=plan_buf)
        out, lse = ops.attn_fwd(g, dv_["q"], dv_["k"], dv_["v"], dsmall["bk"], dsmall["bv"],
                                dv_["coords"], idx.perm, idx.nbr_cl, bias, h, d, workspace=ws, plan=plan)
        fwd_done = torch.cuda.Event()
        fwd_done.record(cur)
        with torch.cuda.stream(s_side):
            s_side.wait_event(fwd_done)
            pooled = ops.merge_pool_fwd(out, dv_["scores"], p_merge, mplan)
            dfe, dsc, _ = ops.merge_pool_bwd(out, dv_["scores"], p_merge, mplan, dv_["dpooled"])
        gr = ops.attn_bwd(g, dv_["q"], dv_["k"], dv_["v"], dsmall["bk"], dsmall["bv"],
                          dv_["coords"], idx, bias, h, d, out, lse, dv_["dout"], workspace=ws, plan=plan)
        cur.wait_stream(s_side)
        outs_d[c] = dict(out=out, lse=lse, dq=gr.dq, dk=gr.dk, dv=gr.dv, pooled=pooled, dfeats=dfe,
                         dscores=dsc)

    # one CUDA graph per chunk (static shapes and buffers): the per-chunk launch cost is a
    # single graph launch, so the chunks can be short and the PCIe fill / drain small
    graphs = [None] * nch
    if not a.no_graph:
        try:
            with torch.cuda.stream(s_cmp):
                for c in range(nch):
                    chunk_compute(c)  # warm-up (allocator, lazy attributes)
            torch.cuda.synchronize()
            for c in range(nch):
                gph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gph, stream=s_cmp):
                    chunk_compute(c)
                graphs[c] = gph
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover - capture is best effort
            print(f"[bench] e2e graph capture failed ({e}); eager chunks", file=sys.stderr)
            graphs = [None] * nch

    def e2e_step():
        ev_in, ev_cmp = [], []
        with torch.cuda.stream(s_in):
            s_in.wait_stream(torch.cuda.current_stream(dev))
            for n in dsmall:
                dsmall[n].copy_(small[n], non_blocking=True)
            for n in dhb:
                dhb[n].copy_(hb[n], non_blocking=True)
            for c, (b0, b1) in enumerate(bounds):
                for n, t in pin.items():
                    dbuf[c][n].copy_(t[b0:b1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
                ev_in.append(e)
        for c, (b0, b1) in enumerate(bounds):
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[c])
                if graphs[c] is not None:
                    graphs[c].replay()
                else:
                    chunk_compute(c)
                e = torch.cuda.Event()
                e.record(s_cmp)
                ev_cmp.append(e)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[c])
                for name, t in outs_d[c].items():
                    outs_h[name][b0:b1].copy_(t, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s_out)

    e2e_step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.e2e_steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    ms = pdist.max_over_ranks(e0.elapsed_time(e1) / a.e2e_steps, dist, dev)
    # PCIe floor of the step: the same byte counts copied H2D and D2H concurrently (pinned)
    hi = torch.empty(int(h2d), dtype=torch.uint8).pin_memory()
    ho = torch.empty(int(d2h), dtype=torch.uint8).pin_memory()
    di = torch.empty(int(h2d), dtype=torch.uint8, device=dev)
    do = torch.empty(int(d2h), dtype=torch.uint8, device=dev)
    floor = []
    for _ in range(3):
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        s_in.wait_stream(torch.cuda.current_stream(dev))
        s_out.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s_in):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s_out):
            ho.copy_(do, non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s_in)
        torch.cuda.current_stream(dev).wait_stream(s_out)
        f1.record()
        torch.cuda.synchronize()
        floor.append(f0.elapsed_time(f1))
    del hi, ho, di, do
    return {"value": B * N * world / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "chunks": nch,
            "pcie_floor_ms": min(floor), "pcie_floor_frac": min(floor) / ms}


# ------------------------------------------------------------- reference
# ------------------------------------------------------------------ pretraining step
def model_flops(cfg, tokens, q):
    """Closed-form flops of one training step per image (BASELINE metric's '% bf16 peak'):
    GEMMs 2*m*n*k forward and twice that backward (dX, dW); attention flop_count_attn
    (proj/src/attention.cpp:360-364) forward and 2.5x that backward (SURVEY §8(d):
    490 D vs 196 D per token)."""
    from paper_2602_16249_b200 import capi
    p2, dd = cfg.patch * cfg.patch, cfg.dec_dim
    gemm, attn = 0, 0
    st = cfg.stages
    gemm += 2 * tokens[0] * (p2 + 16) * st[0].dim
    for s, sc in enumerate(st):
        n, d = tokens[s], sc.dim
        c = -(-n // min(sc.cluster, n))
        width = min(sc.groups, c) * -(-n // c)
        gemm += sc.blocks * 24 * n * d * d
        attn += sc.blocks * capi.flop_count_attn(n, width, sc.heads, d // sc.heads)
        if s + 1 < len(st):
            gemm += 2 * n * d * 16 + 2 * tokens[s + 1] * 2 * d * st[s + 1].dim
            gemm += 2 * q * d * p2  # deep-supervision head
        gemm += 2 * n * (d + 16) * dd  # decoder in-projection + positional MLP
    gemm += 2 * q * 16 * dd + 2 * q * dd * p2
    gemm += len(st) * cfg.dec_depth * 24 * q * dd * dd
    h = cfg.dec_heads
    attn += len(st) * cfg.dec_depth * (capi.flop_count_attn(q, 1, h, dd // h) +
                                       capi.flop_count_attn(q, cfg.self_k, h, dd // h))
    return 3 * gemm + 3.5 * attn, gemm, attn


def run_pretrain(cfg, steps, warmup=3, e2e_steps=6, label="", rank=0, world=1, dist=None):
    """One training step of `cfg` (masks -> encode -> decode -> deep supervision -> loss ->
    backward -> AdamW) through the torch-free model API, captured as one CUDA graph; device
    img/s, plus e2e img/s with the step's images copied H2D from pinned host memory and the
    loss read back D2H inside the timed region."""
    import ctypes as C
    from paper_2602_16249_b200 import capi, devmem
    from paper_2602_16249_b200.model import Model, step_mask_seed
    t0 = time.perf_counter()
    m = Model(cfg)
    create_s = time.perf_counter() - t0
    B = cfg.batch
    if world > 1:  # images shard over ranks; NCCL all-reduce of the gradients inside the step graph
        import torch
        from paper_2602_16249_b200.model import nccl_unique_id
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        m.set_world(world, rank, bytes(idt.cpu().numpy()))
    st = devmem.stream_create()
    L = capi.lib()
    wsb = L.affmae_synth_images_workspace(C.c_int64(B), C.c_int64(cfg.image))
    ws = devmem.DeviceBuffer(wsb)
    seeds = np.arange(400 + rank * B, 400 + (rank + 1) * B, dtype=np.uint64)  # global image index
    capi.check(L.affmae_synth_images(seeds.ctypes.data_as(C.c_void_p), C.c_int64(B), C.c_int64(cfg.image),
                                     C.c_void_p(m.images_ptr), C.c_void_p(ws.ptr), C.c_size_t(wsb), C.c_void_p(st)))
    devmem.sync(st)
    img_bytes = B * cfg.image * cfg.image * 8
    pinned = devmem.PinnedBuffer((B, cfg.image, cfg.image), np.float64)
    pinned.array[...] = devmem.d2h(m.images_ptr, (B, cfg.image, cfg.image), np.float64)
    loss_host = devmem.PinnedBuffer((3,), np.float32)
    step = [0]
    # e2e input pipeline (a data loader's prefetch): step i+1's images go H2D into a device
    # staging buffer on a copy stream while step i computes; each step starts with a D2D copy
    # staging -> the model's input buffer.  Every step's H2D is inside the timed region.
    cs = devmem.stream_create()
    staging = devmem.DeviceBuffer(img_bytes)
    h2d_done, d2d_done = devmem.Event(), devmem.Event()

    def one(e2e=False, prefetch_next=False):
        if e2e:
            devmem.stream_wait(st, h2d_done)  # this step's images landed in staging
            devmem.d2d_async(m.images_ptr, staging.ptr, img_bytes, st)
            d2d_done.record(st)
            if prefetch_next:
                devmem.stream_wait(cs, d2d_done)  # staging free again
                devmem.h2d_async(staging.ptr, pinned.ptr, img_bytes, cs)
                h2d_done.record(cs)
        m.make_masks([step_mask_seed(cfg.seed, (step[0] * world + rank) * B + i) for i in range(B)], stream=st)
        m.train_step(use_graph=True, stream=st, read_loss=False)
        if e2e:
            devmem.d2h_async(loss_host.ptr, m._loss_buf().ptr, 12, st)
        step[0] += 1

    def maxr(v):
        if dist is None:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(warmup):
        one()
    devmem.sync(st)
    if dist is not None:
        dist.barrier()
    e0, e1 = devmem.Event(), devmem.Event()
    e0.record(st)
    for _ in range(steps):
        one()
    e1.record(st)
    e1.synchronize()
    ms = maxr(e0.elapsed_ms(e1) / steps)
    if dist is not None:
        dist.barrier()
    e0.record(st)
    devmem.stream_wait(cs, e0)
    devmem.h2d_async(staging.ptr, pinned.ptr, img_bytes, cs)  # step 0's images (not overlapped)
    h2d_done.record(cs)
    for i in range(e2e_steps):
        one(e2e=True, prefetch_next=i + 1 < e2e_steps)
    e1.record(st)
    e1.synchronize()
    ms_e2e = maxr(e0.elapsed_ms(e1) / e2e_steps)
    loss = devmem.d2h(m._loss_buf().ptr, (3,), np.float32)
    flops, gemm_f, attn_f = model_flops(cfg, m.tokens, m.masked)
    peak = load_bf16_peak()
    tflops = flops * B / (ms * 1e-3) / 1e12
    tflops = tflops * world
    out = {"config": label, "image": cfg.image, "batch_per_gpu": B, "n_gpus": world, "params": int(m.n_values),
           "tokens_per_stage": [int(t) for t in m.tokens], "masked_per_image": int(m.masked),
           "ms_per_step": ms, "img_s": world * B / (ms * 1e-3), "scaling": "weak",
           "grad_allreduce": "ncclAllReduce(sum) of the fp32 gradient arena in the step graph" if world > 1 else None,
           "e2e": {"img_s": world * B / (ms_e2e * 1e-3), "ms_per_step": ms_e2e, "h2d_bytes_per_step": img_bytes,
                   "d2h_bytes_per_step": 12, "steps": e2e_steps,
                   "pipeline": "next step's images H2D on a copy stream during the current step, D2D into the "
                               "model's input buffer at step start; step 0's copy not overlapped"},
           "flops_per_image": flops, "tflops": tflops, "bf16_peak_tflops": peak,
           "frac_bf16_peak": tflops / (peak * world), "loss": [float(x) for x in loss],
           "device_gib": m.device_bytes / 2 ** 30, "create_s": create_s, "cuda_graph": True,
           "step": "masks + encode + decode + deep sup + loss + backward + AdamW (one graph)"}
    m.close()
    pinned.free()
    loss_host.free()
    staging.free()
    return out


def load_bf16_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 2250.0


def ref_pretrain_sample(cfg, threads):
    """The reference's train() (proj/src/pipeline.cpp:682-746) on all host threads, one Model
    replica and one one-step image per thread -> img/s."""
    from oracle import ref
    img = ref.synth_image(cfg.image, 400)
    t0 = time.perf_counter()
    ref.model_train_threads(cfg.c_struct(), threads, 1, img)
    dt = time.perf_counter() - t0
    return threads / dt, dt


# ------------------------------------------------------------- same-run parity
def same_run_parity(a):
    """one image of the timed workload through the same device ops,
    checked against the oracle in this run: index + selection + merge plan bit-exact,
    attention output and dQ/dK/dV rel-L2."""
    import torch
    from oracle import port
    from paper_2602_16249_b200 import ops
    host = make_inputs(argparse.Namespace(**{**vars(a), "batch": 1}), 0)
    dev = torch.device("cuda")
    bf = torch.bfloat16
    t = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device=dev)
    c = host["coords"]
    N = c.shape[1]
    h, d = a.heads, a.head_dim
    geom = ops.geometry(1, N, a.cluster, a.groups)
    idx = ops.cluster_index(t(c, torch.float32), a.cluster, a.groups)
    plan = ops.attn_plan(geom, t(c, torch.float32), idx, h, d, a.hidden)
    bias = ops.BiasNet.from_numpy(host["bias"], device=dev)
    q, k, v, do = (t(host[n], bf) for n in ("q", "k", "v", "dout"))
    bk, bv = t(host["bk"], bf), t(host["bv"], bf)
    out, lse = ops.attn_fwd(geom, q, k, v, bk, bv, t(c, torch.float32), None, None, bias, h, d, plan=plan)
    g = ops.attn_bwd(geom, q, k, v, bk, bv, t(c, torch.float32), idx, bias, h, d, out, lse, do, plan=plan)
    ret = ops.select_retained(t(host["scores"], torch.float32), a.d_s)
    mp = ops.merge_plan(t(c, torch.float32), ret, a.k_m)
    torch.cuda.synchronize()
    ci = port.cluster_index(c[0], a.cluster, a.groups)
    f32 = lambda x: np.asarray(x, np.float32)
    wo = port.attn_fwd(f32(host["q"][0]), f32(host["k"][0]), f32(host["v"][0]), f32(host["bk"]), f32(host["bv"]),
                       c[0], ci["idx"], ci["valid"], host["bias"], h, d)
    wg = port.attn_bwd(f32(host["q"][0]), f32(host["k"][0]), f32(host["v"][0]), f32(host["bk"]), f32(host["bv"]),
                       c[0], ci["idx"], ci["valid"], host["bias"], h, d, f32(host["dout"][0]), prec=32)
    r = port.select_retained(np.asarray(host["scores"][0], np.float64), a.d_s)
    pl = port.merge_plan(c[0], r, a.k_m)

    def rl2(x, y):
        x, y = np.asarray(x, np.float64).ravel(), np.asarray(y, np.float64).ravel()
        return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30))
    res = {"image": 0, "tokens": int(N),
           "index_bit_exact": bool(np.array_equal(idx.perm[0].cpu().numpy(), ci["members"]) and
                                   np.array_equal(idx.nbr_cl[0].cpu().numpy(), ci["nbr_cl"])),
           "retained_bit_exact": bool(np.array_equal(ret[0].cpu().numpy(), r)),
           "merge_plan_bit_exact": bool(np.array_equal(mp.pool_idx[0].cpu().numpy(), pl["pool_idx"]) and
                                        np.array_equal(mp.pool_dist[0].cpu().numpy(), pl["pool_dist"])),
           "attn_out_rel_l2": rl2(out[0].float().cpu().numpy(), wo)}
    for n in ("dq", "dk", "dv"):
        res[f"attn_{n}_rel_l2"] = rl2(getattr(g, n)[0].float().cpu().numpy(), wg[n])
    res["max_rel_l2"] = max(v for kk, v in res.items() if kk.endswith("rel_l2"))
    res["pass"] = bool(res["index_bit_exact"] and res["retained_bit_exact"] and res["merge_plan_bit_exact"]
                       and res["max_rel_l2"] <= 1e-2)
    return res


def ref_sample(a, images, threads):
    """Times oracle/_ref (the unmodified reference, compiled) on `images` images."""
    from oracle import ref
    host = make_inputs(argparse.Namespace(**{**vars(a), "batch": images}), 0)
    f64 = lambda x: np.asarray(x, np.float64)
    t0 = time.perf_counter()
    ref.hotpath_batch(images, threads, 15, host["coords"], f64(host["q"]), f64(host["k"]),
                      f64(host["v"]), f64(host["dout"]), f64(host["scores"]), f64(host["bk"]),
                      f64(host["bv"]), host["bias"], a.heads, a.head_dim, 8.0, a.cluster,
                      a.groups, a.d_s, a.k_m, 1.0)
    dt = time.perf_counter() - t0
    n = host["coords"].shape[1]
    return images * n / dt, dt, n


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_baseline(a):
    from oracle import ref
    if not ref.available():
        return None
    th = host_threads()
    imgs = th  # one image per thread: ~3.5 s of single-core work each at N = 16384
    val, dt, n = ref_sample(a, imgs, th)
    return {"value": val, "unit": UNIT, "cores": th, "kind": "reference",
            "sample": f"{imgs} images x {n} tokens (index + attn fwd+bwd + merge), "
                      f"{th} std::threads, {dt:.1f} s wall"}


def run_reference(a, rank, world):
    """--impl reference: the reference's CPU path on all host threads (rank 0 only)."""
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    th = host_threads()
    for _ in range(a.warmup):
        ref_sample(a, th, th)
    vals, dts = [], []
    n = None
    for _ in range(a.steps):
        v, dt, n = ref_sample(a, th, th)
        vals.append(v)
        dts.append(dt)
    total_tokens = th * n * a.steps
    value = total_tokens / sum(dts)
    cfg = workload_config(a, 1)
    cfg["tokens_per_image"] = n
    cfg["images_per_gpu"] = th
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * sum(dts) / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "reference",
                             "sample": f"{th} images x {n} tokens per step on {th} std::threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def load_traffic(kernel, cfg_key):
    """dram bytes per token from a committed ncu --set full capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t.get(cfg_key, {}).get(kernel)
        return e
    except (OSError, ValueError):
        return None


def run_pretrain_legs(a, rank, world, dist):
    """BASELINE configs[2] (and configs[0]'s shape): the device training step, all ranks."""
    pre = None
    if a.pretrain_batch > 0 or a.tiny_batch > 0:
        from paper_2602_16249_b200.model import aff_tiny, affmae_b
        pre = {}
        try:
            if a.pretrain_batch > 0:
                pre["affmae_b_1024"] = run_pretrain(affmae_b(image=1024, batch=a.pretrain_batch),
                                                    a.pretrain_steps, label="AFFMAE-B 1024^2, 75% mask, deep sup",
                                                    rank=rank, world=world, dist=dist)
            if a.tiny_batch > 0:
                cfg_t = aff_tiny(batch=a.tiny_batch)
                pre["aff_tiny_224"] = run_pretrain(cfg_t, a.pretrain_steps, label="AFF-tiny 224^2, 75% mask",
                                                   rank=rank, world=world, dist=dist)
                if not a.no_cpu_baseline and world == 1:
                    from oracle import ref
                    if ref.available():
                        th = host_threads()
                        v, dt = ref_pretrain_sample(cfg_t, th)
                        pre["aff_tiny_224"]["cpu_reference"] = {
                            "img_s": v, "cores": th, "kind": "reference",
                            "sample": f"{th} images, one train() step each on its own Model replica, {dt:.1f} s"}
                        pre["aff_tiny_224"]["speedup_vs_reference"] = pre["aff_tiny_224"]["img_s"] / v
        except Exception as e:  # pragma: no cover
            pre["error"] = str(e)
    return pre


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        tdist.init_process_group("nccl")
        dist = tdist
    res = run_ours(a, rank, world, dist)
    pre = run_pretrain_legs(a, rank, world, dist)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    N, B = res["N"], res["B"]
    algo = algorithmic_bytes(a, N)
    ph = res["phase_ms"]
    dom = max(("attn_fwd", "attn_bwd"), key=lambda p: ph[p])
    peak, peak_kind = load_peaks()
    achieved = algo[dom] * B * N / (ph[dom] * 1e-3) / 1e9
    cfg_key = f"B{B}_g{a.grid}_D{a.heads * a.head_dim}"
    traffic = load_traffic(dom, cfg_key)
    cfg = workload_config(a, world)
    cfg["tokens_per_image"] = N
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": res["ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": cfg,
        "e2e": {k: v for k, v in res["e2e"].items() if k != "ms_per_step"},
        "gpu_launches": (res["launches"] * a.steps) if res["launches"] else None,
        "roofline": {"kernel": f"{dom} op (all kernels of the C-ABI call)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_token": algo[dom]},
        "phase_ms": ph,
        # every phase against the same HBM roofline (SURVEY §8(d) algorithmic bytes per token)
        "phase_hbm_frac": {k: algo[k] * B * N / (ph[k] * 1e-3) / 1e9 / peak for k in ph if k in algo and ph[k] > 0},
        "clocks": res["clocks"],
        "cuda_graph": res["graph"],
    }
    if res.get("interp"):
        line["next_ops"] = {"interp": res["interp"]}
        if res.get("adamw"):
            line["next_ops"]["adamw"] = res["adamw"]
        if res.get("linear"):
            line["next_ops"]["linear"] = res["linear"]
        if res.get("gattn"):
            line["next_ops"]["decoder_attn"] = res["gattn"]
        if res.get("masks"):
            line["next_ops"]["masks"] = res["masks"]
    # attention tensor flops (flop_count_attn) of the timed step -> fraction of bf16 peak
    from paper_2602_16249_b200 import capi as _capi
    width = res.get("width") or a.cluster * a.groups
    f_fwd = _capi.flop_count_attn(N, width, a.heads, a.head_dim) * B
    bf16_peak = load_bf16_peak()
    line["tensor"] = {"attn_fwd_flops_per_step": f_fwd, "attn_bwd_flops_per_step": 2.5 * f_fwd,
                      "attn_fwd_tflops": f_fwd / (ph["attn_fwd"] * 1e-3) / 1e12,
                      "attn_bwd_tflops": 2.5 * f_fwd / (ph["attn_bwd"] * 1e-3) / 1e12,
                      "frac_bf16_peak_fwd_bwd": 3.5 * f_fwd / ((ph["attn_fwd"] + ph["attn_bwd"]) * 1e-3) / 1e12
                      / bf16_peak, "bf16_peak_tflops": bf16_peak,
                      "note": "HBM-bound op (AI ~25-31 flop/B, SURVEY §0.6): the roofline object is HBM"}
    if not a.no_parity and world == 1:
        try:
            line["parity"] = same_run_parity(a)
        except Exception as e:  # pragma: no cover
            line["parity"] = {"error": str(e)}
    if pre is not None:
        line["pretrain"] = pre
    if not a.no_cpu_baseline and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(a)
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(e)}
    else:
        line["cpu_baseline"] = None
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
