"""CPU multi-process (gloo, world_size 2): image sharding and the max-over-ranks
timing reduction used by bench.py for N > 1 (no data-path collective)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_16249_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    imgs = list(pdist.image_range(4, rank, world))
    seeds = [pdist.mask_seed(i) for i in imgs]
    mx = pdist.max_over_ranks(10.0 + rank, dist)
    sm = pdist.sum_over_ranks(len(imgs), dist)
    q.put((rank, imgs, seeds, mx, sm))
    dist.destroy_process_group()


def test_two_rank_sharding_and_timing_reduce():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    (r0, i0, s0, m0, n0), (r1, i1, s1, m1, n1) = res
    assert i0 == [0, 1, 2, 3] and i1 == [4, 5, 6, 7]          # disjoint global images
    assert s1 == [1004, 1005, 1006, 1007]                      # seeds follow global index
    assert m0 == m1 == 11.0                                    # max over ranks
    assert n0 == n1 == 8.0                                     # all images covered once


def test_single_process_identity():
    assert pdist.max_over_ranks(3.5) == 3.5
    with pytest.raises(ValueError):
        pdist.image_range(4, 2, 2)


def _grad_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.arange(1000, dtype=torch.float32) * (rank + 1)  # rank-dependent gradients
    ar = pdist.GradAllReduce(g, dist, bucket_bytes=1024)       # 256-element buckets
    ar.launch(0, 2)      # early buckets while "backward" continues
    ar.launch(2)         # the rest
    ar.wait()
    q.put((rank, len(ar.buckets), g.numpy().copy()))
    dist.destroy_process_group()


def test_two_rank_bucketed_gradient_allreduce():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_grad_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    (r0, nb0, g0), (r1, nb1, g1) = res
    want = (torch.arange(1000, dtype=torch.float32) * 1.5).numpy()  # mean of 1x and 2x
    assert nb0 == nb1 == 4
    assert (g0 == want).all() and (g1 == want).all()
