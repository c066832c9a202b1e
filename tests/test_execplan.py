"""The executed plan (csrc/host/execplan.hpp) the GPU engine walks, checked on CPU.

It is built from the reference's own planning objects -- build_strategy's PlacementPlan
(placement.hpp:34-63), task_graph (workload.cpp:109-175) and derive_comm_schedule
(placement.hpp:101-102) -- so these tests pin how each placement's
exchanges realise the schedule: every sample is generated once, every scorer sees every
sample of its row set, and every trainer row set ends up with every field of every sample.
"""
import itertools

import pytest

from paper_2312_11819_b200.capi import exec_plan

STRATS = ["colocated", "interleaving1", "interleaving2", "disaggregated"]


def owners(plan, s, r, mb):
    """{sample id: (rank, row)} of row set s for micro-batch (r, mb)."""
    st = plan["sets"][s]
    G, M = plan["G"], plan["micro_batches"]
    Gm, per = G // M, st["per"]
    return {r * G + mb * Gm + i * per + k: (dev, (r * M + mb) * per + k)
            for i, dev in enumerate(st["group"]) for k in range(per)}


def apply(plan, steps):
    """Simulate the exchanges on {(rank, set, field, row): sample id} and return the state."""
    have = {}
    B, G = plan["batch_per_rank"], plan["G"]
    for r in range(plan["rollouts"]):
        for k in range(plan["world"]):
            for b in range(B):
                have[(k, -1, "prompt", r * B + b)] = r * G + k * B + b
    field_of = {"Actor": "logp_old", "ShadowActor": "logp_old", "Ref": "logp_ref", "Critic": "values",
                "ShadowCritic": "values", "Reward": "score"}
    for st in steps:
        if st["kind"] == "exchange":
            for mv in st["moves"]:
                f = mv["field"]
                for src, dst, srow, drow, cnt in mv["transfers"]:
                    for q in range(cnt):
                        v = have[(src, mv["src_set"], f, srow + q)]
                        have[(dst, mv["dst_set"], "tokens" if f == "prompt" else f, drow + q)] = v
        elif st["kind"] == "task":
            t = plan["tasks"][st["task"]]
            if t["kind"] in ("Generation", "Forward"):
                s = plan["set_of"][t["model"]]
                for sid, (dev, row) in owners(plan, s, t["rollout"], t["mb"]).items():
                    assert have.get((dev, s, "tokens", row)) == sid, (t, sid)  # input rows present
                    if t["kind"] == "Forward":
                        have[(dev, s, field_of[t["model"]], row)] = sid
    return have


@pytest.mark.parametrize("strategy,world,mb,ro", [(s, w, mb, ro) for s in STRATS for w in (1, 2, 4)
                                                  for mb, ro in ((1, 1), (2, 1), (2, 2)) if not (w == 1 and s != "colocated")])
def test_exchanges_deliver_every_field_to_every_trainer(strategy, world, mb, ro):
    B = 4
    plan = exec_plan(strategy, world, B, 16, 16, micro_batches=mb, rollout_nums=ro)
    have = apply(plan, plan["steps"])
    for model in ("Actor", "Critic"):
        s = plan["set_of"][model]
        for r, m in itertools.product(range(ro), range(mb)):
            for sid, (dev, row) in owners(plan, s, r, m).items():
                for f in ("tokens", "logp_old", "logp_ref", "values", "score"):
                    assert have.get((dev, s, f, row)) == sid, (model, f, sid)


@pytest.mark.parametrize("strategy", STRATS)
def test_generation_runs_once_per_sample(strategy):
    plan = exec_plan(strategy, 2, 4, 16, 16, micro_batches=2, rollout_nums=2)
    gen = plan["generator"]
    s = plan["set_of"][gen]
    seen = []
    for t in plan["tasks"]:
        if t["kind"] == "Generation":
            seen += list(owners(plan, s, t["rollout"], t["mb"]))
    assert sorted(seen) == list(range(2 * 2 * 4))


def test_colocated_single_gpu_has_only_local_prompt_copies():
    plan = exec_plan("colocated", 1, 4, 16, 16)
    kinds = [s["kind"] for s in plan["steps"]]
    assert kinds == ["exchange", "task", "exchange", "task", "task", "task", "task", "exchange", "experience", "task",
                     "optimizer_step", "task", "optimizer_step"]
    for st in plan["steps"]:
        for mv in st["moves"]:
            assert mv["field"] == "prompt" and all(t[0] == t[1] for t in mv["transfers"])
    assert plan["comm_ops"] == []


def test_interleaving_exchanges_realise_allgather_and_alltoall():
    """Alg. 1: AllGather of (query, response) before the Ref/Reward forwards, AlltoAll of the
    outputs after -- the exchange steps carry those CommOps."""
    plan = exec_plan("interleaving1", 2, 4, 16, 16)
    ops = plan["comm_ops"]
    ex = [s for s in plan["steps"] if s["kind"] == "exchange" and s["comm_op"] >= 0]
    assert sorted(ops[s["comm_op"]]["kind"] for s in ex) == ["AllGather", "AlltoAll"]
    before = next(s for s in ex if ops[s["comm_op"]]["kind"] == "AllGather")
    # Ref on {0}, Reward on {1}: each receives the other rank's generated tokens
    assert {(t[0], t[1]) for mv in before["moves"] for t in mv["transfers"]} >= {(1, 0), (0, 1)}


def test_disaggregated_sends_experience_to_trainers_and_syncs_params():
    plan = exec_plan("disaggregated", 2, 4, 16, 16, micro_batches=2)
    assert plan["generator"] == "ShadowActor"
    trn, inf = plan["set_of"]["Actor"], plan["set_of"]["ShadowActor"]
    assert plan["sets"][trn]["group"] == [0] and plan["sets"][inf]["group"] == [1]
    after = [s for s in plan["steps"] if s["kind"] == "exchange" and s["attach"] == "after"]
    assert len(after) == 2  # one per micro-batch (Alg. 2: Send outputs to the training devices)
    fields = {mv["field"] for mv in after[0]["moves"]}
    assert fields == {"tokens", "logp_old", "logp_ref", "values", "score"}
    assert all(t[0] == 1 and t[1] == 0 for mv in after[0]["moves"] for t in mv["transfers"])
    syncs = [t for t in plan["tasks"] if t["kind"] == "ParamSync"]
    assert [t["model"] for t in syncs] == ["ShadowActor", "ShadowCritic"]


def test_ppo_epochs_and_optimizer_steps():
    plan = exec_plan("colocated", 1, 4, 16, 16, micro_batches=2, ppo_epochs=3)
    opt = [(s["model"], s["epoch"]) for s in plan["steps"] if s["kind"] == "optimizer_step"]
    assert opt == [(m, e) for e in range(3) for m in ("Actor", "Critic")]
    trains = [t for t in plan["tasks"] if t["kind"] == "TrainFB"]
    assert len(trains) == 2 * 2 * 3


def test_ratio_vector_placement_executes_any_grouping():
    """PlacementRatioVector (placement.hpp:29-46): Actor/Critic on all 4, Ref on half, Reward on a quarter."""
    plan = exec_plan("ratio_vector", 4, 4, 16, 16, ratios=(1.0, 1.0, 0.5, 0.25))
    assert len(plan["sets"][plan["set_of"]["Ref"]]["group"]) == 2
    assert len(plan["sets"][plan["set_of"]["Reward"]]["group"]) == 1
    have = apply(plan, plan["steps"])
    s = plan["set_of"]["Actor"]
    for sid, (dev, row) in owners(plan, s, 0, 0).items():
        assert have.get((dev, s, "score", row)) == sid


def test_indivisible_split_is_a_config_error():
    with pytest.raises(RuntimeError, match="error 2"):
        exec_plan("interleaving1", 4, 1, 16, 16, micro_batches=4)  # 1 sample per micro-batch over 2 Ref devices
