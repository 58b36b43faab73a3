"""Data-parallel training step: a 2-rank step over images {0, 1} | {2, 3}
(gloo, world size 2, both ranks on the one GPU of the test box, gradients summed host-side
between forward_backward and apply_step) equals the 1-rank step over images {0, 1, 2, 3}:
the loss gradient is seeded with 1/world, so the summed gradient is the global batch mean.
Images and mask seeds follow the GLOBAL image index, so results do not depend on the split."""
import os
import socket

import numpy as np
import pytest

from oracle import ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _cfg(batch):
    from tests.test_model_gpu import small_cfg
    return small_cfg(batch=batch, warmup=2, total_steps=4)


def _inputs(global_ids):
    from paper_2602_16249_b200.model import step_mask_seed
    imgs = np.stack([ref.synth_image(64, 500 + i) for i in global_ids])
    seeds = [step_mask_seed(1, i) for i in global_ids]
    return imgs, seeds


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2602_16249_b200.model import Model
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = Model(_cfg(2))
    m.set_world(world, rank)
    imgs, seeds = _inputs([2 * rank, 2 * rank + 1])
    m.set_images(imgs)
    m.make_masks(seeds)
    m.forward_backward()
    g = torch.from_numpy(m.grads_device_to_host())
    dist.all_reduce(g)  # the step's one exchange (NCCL on multi-GPU boxes, gloo here)
    m.grads_host_to_device(g.numpy())
    np.save(os.path.join(out_dir, f"grads{rank}.npy"), g.numpy())
    m.apply_step()
    p = m.params()
    np.savez(os.path.join(out_dir, f"params{rank}.npz"), **p)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_step_equals_one_rank_step(tmp_path):
    import torch.multiprocessing as mp
    from paper_2602_16249_b200.model import Model
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    one = Model(_cfg(4))
    imgs, seeds = _inputs([0, 1, 2, 3])
    one.set_images(imgs)
    one.make_masks(seeds)
    one.forward_backward()
    g1 = one.grads_device_to_host()
    g2 = np.load(tmp_path / "grads0.npy")
    np.testing.assert_array_equal(g2, np.load(tmp_path / "grads1.npy"))  # every rank holds the same sum
    rel = np.linalg.norm(g2 - g1) / np.linalg.norm(g1)
    assert rel <= 1e-4, rel
    one.apply_step()
    p1 = one.params()
    p2 = dict(np.load(tmp_path / "params0.npz"))
    lr = 1e-3 * 1 / 2  # warmup 2: lr_at(0) = lr / 2
    worst = max(float(np.abs(p1[n] - p2[n]).max()) for n in p1)
    assert worst <= 2.0 * lr + 1e-7, worst  # an element whose tiny gradient flips sign moves by <= 2 lr
    frac = np.mean(np.concatenate([(np.abs(p1[n] - p2[n]) <= 1e-6).ravel() for n in p1]))
    assert frac >= 0.999, frac


def test_nccl_exchange_in_the_step_graph_single_rank():
    """The NCCL path of the step (runtime-loaded libnccl, communicator init, ncclAllReduce of the
    gradient arena captured in the step's CUDA graph) on a one-rank communicator -- the only
    NCCL topology a one-GPU box offers: the sum over one rank is the identity, so the step
    equals the step without a communicator (to the step's own run-to-run rounding: the
    reverse-CSR fills are order-nondeterministic, see test_graph_replay_matches_eager)."""
    from paper_2602_16249_b200.model import Model, nccl_unique_id
    imgs, seeds = _inputs([0, 1])
    out = []
    for use_nccl in (False, True):
        m = Model(_cfg(2))
        if use_nccl:
            m.set_world(1, 0, nccl_unique_id())
        m.set_images(imgs)
        m.make_masks(seeds)
        m.train_step()
        m.make_masks(seeds)
        m.train_step()
        out.append(m.params())
        m.close()
    worst = max(float(np.abs(out[0][n] - out[1][n]).max()) for n in out[0])
    assert worst <= 4e-3, worst  # 2 steps, an element whose tiny gradient flips sign moves <= 2 lr
    frac = np.mean(np.concatenate([(np.abs(out[0][n] - out[1][n]) <= 1e-6).ravel() for n in out[0]]))
    assert frac >= 0.99, frac
