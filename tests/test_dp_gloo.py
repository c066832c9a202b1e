"""Multi-rank host logic on CPU (world_size 2, gloo): the Co-located data-parallel
split the engine uses at N GPUs.

Each rank takes samples [rank*Bg, (rank+1)*Bg) (rlhf_ppo_config.sample_offset)
and scales its loss by the GLOBAL B*R (loss_denominator); the gradient
all-reduce (NCCL on the GPU path, gloo here) must then reproduce the full-batch
gradient and loss of a single-process step.  Compute runs in the CPU oracle.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_11819_b200.capi import make_config

B, P, R, WORLD = 4, 16, 16, 2


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from tests import oracle_lib
    bg = B // WORLD
    cfg = make_config("tiny", "tiny", bg, P, R, sample_offset=rank * bg, loss_denominator=float(B * R))
    o = oracle_lib.ppo_step(cfg, threads=2)
    g = torch.from_numpy(np.concatenate([o["actor_grad"], o["critic_grad"]]))
    loss = torch.tensor([o["actor_loss"], o["critic_loss"]], dtype=torch.float64)
    dist.all_reduce(g)
    dist.all_reduce(loss)
    toks = [torch.zeros(bg, P + R, dtype=torch.int32) for _ in range(WORLD)]
    dist.all_gather(toks, torch.from_numpy(o["tokens"]))
    if rank == 0:
        out.put((g.numpy(), loss.numpy(), torch.cat(toks).numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_data_parallel_matches_single_process():
    from tests import oracle_lib
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    g, loss, toks = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    full = oracle_lib.ppo_step(make_config("tiny", "tiny", B, P, R), threads=2)
    np.testing.assert_array_equal(toks, full["tokens"])  # sharded generation == full-batch generation
    ref = np.concatenate([full["actor_grad"], full["critic_grad"]])
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) < 1e-4
    np.testing.assert_allclose(loss, [full["actor_loss"], full["critic_loss"]], rtol=1e-4)
