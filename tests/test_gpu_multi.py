"""Placement strategies on 2 GPUs vs the full-batch CPU oracle (needs >= 2 GPUs).

Each rank owns a prompt shard of Bg samples (global ids rank*Bg + b).  Whatever
placement executes the step -- Co-located data parallel, Interleaving1 (Ref |
Reward split, token AllGather + output AlltoAll), Interleaving2 (Actor+Ref |
Critic+Reward), Disaggregated (trainers | shadow-actor inference + ParamSync) --
the union of the ranks' experience rows, the all-reduced gradients and the
updated weights must equal one full-batch PPO step ("synchronous
training without compromising model accuracy" made exact).  Tolerances as in
tests/test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

from paper_2312_11819_b200.capi import make_config, named_slices

pytestmark = pytest.mark.gpu

BG, P, R, WORLD = 2, 16, 16, 2


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _rank(rank, strategy, q_id, q_out, zero=0, arch="tiny"):
    import torch
    torch.cuda.set_device(rank)
    from paper_2312_11819_b200.capi import make_config as mc
    from paper_2312_11819_b200.engine import Engine
    if rank == 0:
        nid = Engine.nccl_unique_id()
        for _ in range(WORLD - 1):
            q_id.put(nid)
    else:
        nid = q_id.get(timeout=120)
    cfg = mc(arch, arch, BG, P, R, sample_offset=rank * BG, loss_denominator=float(BG * WORLD * R))
    eng = Engine(cfg, device=rank, rank=rank, world_size=WORLD, strategy=strategy, nccl_id=nid, zero_stage=zero)
    eng.step()
    out = {"rank": rank, "sample_ids": eng.read("sample_ids")}
    for k in ("tokens", "logp_old", "logp_ref", "values", "score", "advantages", "returns", "actor_grad", "critic_grad",
              "actor_master", "critic_master", "actor_params", "shadow_actor_params", "shadow_critic_params",
              "critic_params"):
        try:
            out[k] = eng.read(k)
        except Exception:
            pass
    q_out.put(out)


@pytest.fixture(scope="module")
def oracle():
    from tests import oracle_lib
    return oracle_lib


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("strategy", ["colocated", "interleaving1", "interleaving2", "disaggregated"])
def test_two_gpu_placement_matches_full_batch_oracle(strategy, oracle):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_id, q_out = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, strategy, q_id, q_out)) for r in range(WORLD)]
    for p in procs:
        p.start()
    outs = [q_out.get(timeout=600) for _ in range(WORLD)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    B = BG * WORLD
    # assemble experience rows by global sample id
    tokens = np.zeros((B, P + R), np.int32)
    got = {k: {} for k in ("logp_old", "logp_ref", "values", "score", "advantages", "returns")}
    for o in outs:
        for row, sid in enumerate(o["sample_ids"]):
            if sid < 0 or "tokens" not in o:
                continue
            tokens[sid] = o["tokens"][row]
            for k in got:
                if k in o and (k != "score"):
                    got[k][sid] = o[k][row]
                elif k in o:
                    got[k][sid] = o[k][row]
    assert all(len(v) == B for v in got.values()), {k: len(v) for k, v in got.items()}
    cfg = make_config("tiny", "tiny", B, P, R)
    ora = oracle.ppo_step(cfg, tokens_in=tokens)
    m = ora["greedy_margin"] > 1e-2
    np.testing.assert_array_equal(tokens[:, P:][m], ora["greedy_pred"][m])
    for k, atol in (("logp_old", 2e-2), ("logp_ref", 2e-2), ("values", 2e-2), ("score", 2e-2), ("advantages", 5e-2),
                    ("returns", 5e-2)):
        mine = np.stack([got[k][s] for s in range(B)])
        np.testing.assert_allclose(mine, ora[k], atol=atol, rtol=1e-3, err_msg=f"{strategy}:{k}")
    for tag in ("actor", "critic"):
        holders = [o for o in outs if f"{tag}_grad" in o]
        assert holders, f"no rank trains the {tag}"
        arch = cfg.actor if tag == "actor" else cfg.critic
        for o in holders:
            g, go = o[f"{tag}_grad"], ora[f"{tag}_grad"]
            for name, off, n in named_slices(arch):
                a, b = g[off:off + n].astype(np.float64), go[off:off + n].astype(np.float64)
                err = np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12)
                assert err <= 3e-2, (strategy, tag, name, err)
            lr = 1e-5 if tag == "actor" else 5e-6
            assert np.abs(o[f"{tag}_master"] - ora[f"{tag}_master"]).max() <= 2 * lr + 1e-7
    if strategy == "disaggregated":  # ParamSync: shadows hold the trainers' updated bf16 weights
        trainer = next(o for o in outs if "actor_params" in o)
        inference = next(o for o in outs if "shadow_actor_params" in o)
        np.testing.assert_array_equal(inference["shadow_actor_params"], trainer["actor_params"])
        np.testing.assert_array_equal(inference["shadow_critic_params"], trainer["critic_params"])


def _spawn(strategy, zero, arch):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_id, q_out = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, strategy, q_id, q_out, zero, arch)) for r in range(WORLD)]
    for p in procs:
        p.start()
    outs = sorted((q_out.get(timeout=600) for _ in range(WORLD)), key=lambda o: o["rank"])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return outs


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("arch", ["tiny", "llama-tiny"])
def test_zero1_sharded_adamw_is_bit_identical_to_replicated(arch):
    """ZeRO-1 (reduce-scatter of gradients, AdamW on a 1/dp slice of master/m/v, all-gather of
    the bf16 weights) against the replicated all-reduce step on the same data-parallel pair:
    the sum of two addends is order-free, so updated weights and master slices match bit for bit."""
    from paper_2312_11819_b200.capi import param_total
    z0, z1 = _spawn("colocated", 0, arch), _spawn("colocated", 1, arch)
    cfg = make_config(arch, arch, BG, P, R)
    for tag, a in (("actor", cfg.actor), ("critic", cfg.critic)):
        n = param_total(a)
        shard = ((n + WORLD - 1) // WORLD + 63) // 64 * 64
        for r in range(WORLD):
            np.testing.assert_array_equal(z1[r][f"{tag}_params"], z0[r][f"{tag}_params"], err_msg=f"{tag} rank {r}")
            m1 = z1[r][f"{tag}_master"]
            assert m1.size == shard
            lo, hi = r * shard, min(n, (r + 1) * shard)
            np.testing.assert_array_equal(m1[:hi - lo], z0[r][f"{tag}_master"][lo:hi])
            assert not m1[hi - lo:].any()


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("arch", ["tiny", "llama-tiny"])
def test_zero2_bucket_sharded_gradients_match_replicated(arch):
    """ZeRO-2 (per-layer gradient buckets reduce-scattered on the comm stream during the
    backward, AdamW on each rank's bucket slices, bf16 slices all-gathered) against the
    replicated all-reduce step: the gradient sums associate differently (per bucket, per
    chunk), so updated weights agree to the first AdamW step's sign-like contract."""
    z0, z2 = _spawn("colocated", 0, arch), _spawn("colocated", 2, arch)
    for tag, lr in (("actor", 1e-5), ("critic", 5e-6)):
        for r in range(WORLD):
            a = z0[r][f"{tag}_params"].view(np.uint16).astype(np.uint32) << 16
            b = z2[r][f"{tag}_params"].view(np.uint16).astype(np.uint32) << 16
            fa, fb = a.view(np.float32), b.view(np.float32)
            assert (np.abs(fa - fb) <= 2 * lr + np.abs(fa) * 2 ** -7).all(), tag  # a flip or one bf16 ulp
            assert np.mean(fa != fb) <= 1e-3, (tag, np.mean(fa != fb))
        np.testing.assert_array_equal(z2[0][f"{tag}_params"], z2[1][f"{tag}_params"])  # replicas agree


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("zero", [2, 3])
def test_disaggregated_zero23_paramsync_matches_replicated(zero):
    """Disaggregated trainers under ZeRO-2 (bucket-sharded gradients) and ZeRO-3 (weights
    sharded too: each decoder layer all-gathered on the comm stream as it runs, ParamSync
    all-gathers bucket by bucket and broadcasts to the shadows) against ZeRO-0: the shadows
    receive the same updated weights (one trainer per group here, so the bucket slices are
    whole buckets and the arithmetic is the replicated one)."""
    z0, zz = _spawn("disaggregated", 0, "tiny"), _spawn("disaggregated", zero, "tiny")
    inf0 = next(o for o in z0 if "shadow_actor_params" in o)
    infz = next(o for o in zz if "shadow_actor_params" in o)
    for key in ("shadow_actor_params", "shadow_critic_params"):
        a, b = inf0[key], infz[key]
        assert np.mean(a != b) <= 1e-4, (key, np.mean(a != b))
