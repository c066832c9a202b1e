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


# ---- every placement's exchange logic, executed on CPU ranks over gloo ------------------
# The GPU engine walks csrc/host/execplan.hpp's plan (rank roles, per-model sample
# partitions, row transfers at each exchange).  Here the SAME plan (through the C-ABI) is
# executed by world-size-2 gloo ranks: the oracle computes each task on the rank's own row
# block, rows move by gloo send/recv exactly as the plan lists them, each trained model's
# gradient is all-reduced over its device group.  The union of experience rows and the
# reduced gradients must equal ONE full-batch oracle step (synchronous
# training without compromising model accuracy).
PB, PP, PR = 2, 16, 16  # per-rank batch, prompt, response (tiny decoder)


def _owners(plan, s, r, mb):
    st = plan["sets"][s]
    G, M = plan["G"], plan["micro_batches"]
    per = st["per"]
    return [(r * G + mb * (G // M) + i * per, dev, (r * M + mb) * per) for i, dev in enumerate(st["group"])]


def _placement_worker(rank, port, strategy, mb, ro, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2312_11819_b200.capi import exec_plan, prompt_tokens
    from tests import oracle_lib
    plan = exec_plan(strategy, WORLD, PB, PP, PR, micro_batches=mb, rollout_nums=ro)
    S, G = PP + PR, plan["G"]
    groups = {m: dist.new_group(plan["sets"][plan["set_of"][m]]["group"]) for m in ("Actor", "Critic")}
    field_of = {"Actor": "logp_old", "ShadowActor": "logp_old", "Ref": "logp_ref", "Critic": "values",
                "ShadowCritic": "values", "Reward": "score"}
    bufs = {}
    for si, st in enumerate(plan["sets"]):
        if rank in st["group"]:
            n = st["rows"]
            bufs[si] = dict(tokens=np.zeros((n, S), np.int32), logp_old=np.zeros((n, PR), np.float32),
                            logp_ref=np.zeros((n, PR), np.float32), values=np.zeros((n, PR), np.float32),
                            score=np.zeros(n, np.float32))
    home = np.zeros((ro * PB, S), np.int32)
    cfg0 = make_config("tiny", "tiny", 1, PP, PR)
    for r in range(ro):
        home[r * PB:(r + 1) * PB, :PP] = prompt_tokens(cfg0.prompt_seed, PB, PP, cfg0.actor.vocab,
                                                       sample_offset=r * G + rank * PB)
    grads = {}
    for st in plan["steps"]:
        if st["kind"] == "exchange":
            sends, recvs = [], []
            for mv in st["moves"]:
                f = "tokens" if mv["field"] == "prompt" else mv["field"]
                src = home if mv["src_set"] < 0 else (bufs[mv["src_set"]][f] if mv["src_set"] in bufs else None)
                dst = bufs.get(mv["dst_set"], {}).get(f)
                for s_, d_, sr, dr, c in mv["transfers"]:
                    if s_ == rank and d_ == rank:
                        dst[dr:dr + c] = src[sr:sr + c]
                    elif s_ == rank:
                        sends.append(dist.isend(torch.from_numpy(np.ascontiguousarray(src[sr:sr + c])), d_))
                    elif d_ == rank:
                        t = torch.from_numpy(np.zeros_like(dst[dr:dr + c]))
                        recvs.append((dist.irecv(t, s_), t, dst, dr, c))
            for q in sends:
                q.wait()
            for q, t, dst, dr, c in recvs:
                q.wait()
                dst[dr:dr + c] = t.numpy()
        elif st["kind"] == "task":
            t = plan["tasks"][st["task"]]
            m = t["model"]
            if t["kind"] in ("Generation", "Forward") and m in plan["set_of"]:
                s = plan["set_of"][m]
                for first, dev, row0 in _owners(plan, s, t["rollout"], t["mb"]):
                    if dev != rank:
                        continue
                    per = plan["sets"][s]["per"]
                    blk = bufs[s]["tokens"][row0:row0 + per]
                    cfg = make_config("tiny", "tiny", per, PP, PR, sample_offset=first)
                    if t["kind"] == "Generation":
                        o = oracle_lib.ppo_step(cfg, stop_after=1, threads=1)
                        assert np.array_equal(o["tokens"][:, :PP], blk[:, :PP]), "prompt exchange delivered wrong rows"
                        blk[:] = o["tokens"]
                    else:
                        o = oracle_lib.ppo_step(cfg, tokens_in=blk, stop_after=1, threads=1)
                        bufs[s][field_of[m]][row0:row0 + per] = o[field_of[m]]
            elif t["kind"] == "TrainFB" and t["mb"] == 0 and t["epoch"] == 0 and rank in \
                    plan["sets"][plan["set_of"][m]]["group"]:
                # this rank's gradient share: its trainer rows, loss over the GLOBAL G * R
                b = bufs[plan["set_of"][m]]
                cfg = make_config("tiny", "tiny", len(b["tokens"]), PP, PR, loss_denominator=float(G * ro * PR))
                o = oracle_lib.ppo_step(cfg, tokens_in=b["tokens"], threads=1)
                g = torch.from_numpy(o["actor_grad" if m == "Actor" else "critic_grad"].copy())
                dist.all_reduce(g, group=groups[m])
                grads[m] = g.numpy()
    # experience rows held by this rank (Actor's trainer set, else Critic's): by sample id
    es = plan["set_of"]["Actor"] if rank in plan["sets"][plan["set_of"]["Actor"]]["group"] else plan["set_of"]["Critic"]
    rows = {}
    st = plan["sets"][es]
    for r in range(ro):
        for m_ in range(mb):
            for first, dev, row0 in _owners(plan, es, r, m_):
                if dev == rank:
                    for k in range(st["per"]):
                        rows[first + k] = {f: bufs[es][f][row0 + k].copy() for f in bufs[es]}
    out.put((rank, rows, grads))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("strategy,mb,ro", [("colocated", 1, 1), ("interleaving1", 1, 1), ("interleaving2", 2, 1),
                                            ("disaggregated", 2, 1), ("interleaving1", 2, 2), ("disaggregated", 1, 2)])
def test_placement_exchanges_over_gloo_match_single_process(strategy, mb, ro):
    from tests import oracle_lib
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() * 7 + hash(strategy) + mb * 13 + ro) % 900
    procs = [ctx.Process(target=_placement_worker, args=(r, port, strategy, mb, ro, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    G = WORLD * PB * ro
    full = oracle_lib.ppo_step(make_config("tiny", "tiny", G, PP, PR), threads=2)
    seen = set()
    for _, rows, _ in res:
        for sid, f in rows.items():
            seen.add(sid)
            np.testing.assert_array_equal(f["tokens"], full["tokens"][sid])
            for k in ("logp_old", "logp_ref", "values", "score"):
                np.testing.assert_allclose(f[k], full[k][sid], atol=1e-5, err_msg=f"{strategy}: {k} of sample {sid}")
    assert seen == set(range(G))
    for m, key in (("Actor", "actor_grad"), ("Critic", "critic_grad")):
        holders = [g[m] for _, _, g in res if m in g]
        assert holders, f"no rank trains the {m}"
        for g in holders:
            assert np.linalg.norm(g - full[key]) / np.linalg.norm(full[key]) < 1e-4, (strategy, m)
