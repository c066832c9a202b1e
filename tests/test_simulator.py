"""The planner/simulator path (csrc/host/simulator.cpp, costmodel.cpp) against the
reference's specification: /root/reference/SPEC.md acceptance criteria 1-3, 8, 10, 11 and
the costmodel / simulator / planner examples.  Pure host logic."""
import json

import pytest

from paper_2312_11819_b200.capi import sim_run

A100_1x8 = {"groups": [{"nodes": 1, "devices_per_node": 8, "kind": "A100", "memory_GB": 80, "peak_TFLOPs": 312,
                        "hbm_GBps": 2000}], "intra_node_GBps": 600, "inter_node_GBps": 100, "inter_type_GBps": 25}


def topo(nodes, per=8):
    t = json.loads(json.dumps(A100_1x8))
    t["groups"][0]["nodes"] = nodes
    t["groups"][0]["devices_per_node"] = per
    return t


def scen(sizes, strategies, batch=8, nodes=1, per=8, **kw):
    s = {"topology": topo(nodes, per),
         "workload": {"sizes_B": {"actor": sizes[0], "critic": sizes[1], "ref": sizes[2], "reward": sizes[3]},
                      "batch": batch, **kw.pop("workload", {})},
         "strategies": strategies}
    s.update(kw)
    return s


def sim(s):
    return sim_run("simulate", s)


def test_oom_reproduction_65b_vs_7b():
    """Acceptance 3 (Table I): 65B AC-NonShare Co-located on 1x8x80 GB is infeasible (exit
    code 3).  The spec's memory model replicates the inference-only Ref/Reward at 2 B/param on
    every device (ZeRO applies to trainable models only), which puts 13B at
    4 x 26 GB > 76 GB; 7B is the feasible row under those constants."""
    big = scen((65, 65, 65, 65), [{"name": "colocated", "zero_level": 3, "batch": 8}])
    with pytest.raises(RuntimeError, match="error 3"):
        sim(big)
    small = scen((7, 7, 7, 7), [{"name": "colocated", "zero_level": 3, "batch": 8}])
    assert sim(small)["feasible"]


def test_max_batch_interleaving_at_least_colocated():
    """Acceptance 8: freed redundancy only adds headroom."""
    s = scen((7, 7, 7, 7), [{"name": "colocated", "zero_level": 3}, {"name": "interleaving1", "zero_level": 3}])
    mb = {r["name"]: r["max_batch"] for r in sim_run("maxbatch", s)}
    assert mb["interleaving1"] >= mb["colocated"] > 0


def test_simulator_invariants():
    """Acceptance 10: conservation lower bound, overlap dominance, bubble monotone in
    micro-batches under Disaggregated, ParamSync before the next Generation, determinism."""
    base = scen((7, 7, 7, 7), [{"name": "disaggregated", "zero_level": 2, "tp_gen": 4, "batch": 32}], nodes=2,
                workload={"micro_batches": 1})
    r = sim(base)
    for d, busy in r["per_device_busy_seconds"].items():
        assert r["step_seconds"] >= busy - 1e-9
    off = json.loads(json.dumps(base))
    off["sim"] = {"overlap": False}
    assert sim(base)["step_seconds"] <= sim(off)["step_seconds"] + 1e-12
    bubbles = []
    for k in (1, 2, 4, 8):
        s = json.loads(json.dumps(base))
        s["workload"]["micro_batches"] = k
        bubbles.append(sim(s)["bubble_fraction"])
    assert all(b2 <= b1 + 1e-5 for b1, b2 in zip(bubbles, bubbles[1:])), bubbles  # (alpha per extra message)
    assert bubbles[-1] < bubbles[0]
    tr = json.loads(json.dumps(base))
    tr["sim"] = {"iterations": 2}
    trace = sim_run("trace", tr)
    ev = [e for e in trace["traceEvents"] if e["ph"] == "X"]
    syncs = [e for e in ev if e["name"].startswith("sync:")]
    gens = sorted(e["ts"] for e in ev if e["name"].startswith("generation:"))
    first_sync_end = min(e["ts"] + e["dur"] for e in syncs)
    assert any(g >= first_sync_end for g in gens)  # iteration 2 generates after the ParamSync
    assert all(sim_run("trace", tr) == trace for _ in range(3))  # byte-stable
    assert sim(base) == r


def test_stage_fractions_partition_the_step():
    r = sim(scen((7, 7, 7, 7), [{"name": "interleaving1", "zero_level": 3, "batch": 16}]))
    assert abs(sum(r["per_stage_fraction"].values()) - 1.0) < 1e-6
    assert r["throughput_samples_per_sec"] > 0
    assert r["busiest_stage"] == max(r["per_stage_seconds"], key=r["per_stage_seconds"].get)


def test_generation_dominates_colocated_33b_with_default_constants():
    """costmodel example: 33B Co-located with the default MFUs -> Generation >= 85 %."""
    s = scen((33, 33, 33, 33), [{"name": "colocated", "zero_level": 3, "batch": 16}], nodes=4,
             sim={"allow_infeasible": True})
    assert sim(s)["per_stage_fraction"]["generation"] >= 0.85


def test_calibrate_single_observation_is_exact_and_idempotent():
    """calibrate (costmodel.hpp:78-90): one observation -> exact fit; duplicates -> same result."""
    s = scen((7, 7, 7, 7), [{"name": "colocated", "zero_level": 3, "batch": 16}])
    ob = {"strategy": {"name": "colocated", "zero_level": 3}, "devices": 8, "batch": 16,
          "measured_step_seconds": 40.0, "generation_fraction": 0.9}
    c1 = sim_run("calibrate", {"scenario": s, "observations": [ob]})
    o = c1["observations"][0]
    assert abs(o["predicted_step_seconds"] - 40.0) / 40.0 < 1e-6
    assert abs(o["predicted_per_stage_fraction"]["generation"] - 0.9) < 1e-6
    c2 = sim_run("calibrate", {"scenario": s, "observations": [ob, ob]})
    assert c1["constants"] == c2["constants"]
    with pytest.raises(RuntimeError, match="error 2"):
        sim_run("calibrate", {"scenario": s, "observations": [dict(ob, measured_step_seconds=0.0)]})


def test_strict_scenario_parser():
    with pytest.raises(RuntimeError, match="unknown key"):
        sim(scen((1, 1, 1, 1), [{"name": "colocated", "batch": 4, "zero": 1}]))
    with pytest.raises(RuntimeError, match="line"):
        sim_run("simulate", '{"workload": {"batch": 4,}}')


def test_compare_sorted_and_oom_rows_last():
    s = scen((65, 65, 65, 65), [{"name": "colocated", "zero_level": 3, "batch": 8},
                                {"name": "interleaving2", "zero_level": 3, "batch": 8}], nodes=2)
    out = sim_run("compare", s)
    rows = out["rows"]
    feas = [r["feasible"] for r in rows]
    assert feas == sorted(feas, reverse=True)
    thr = [r["throughput"] for r in rows if r["feasible"]]
    assert thr == sorted(thr, reverse=True)
    assert out["csv"].startswith("strategy,feasible,max_batch")
    assert "OOM" in out["table"] or all(feas)


def test_recommend_rules():
    """Planner rule 1 (example :468): 1x8, 7B, Ref fits one node -> Interleaving;
    rule 2 (> 2 nodes) -> Disaggregated with inference share in [0.3, 0.5]."""
    r = sim_run("plan", scen((7, 7, 7, 7), []))
    assert r["strategy"].startswith("interleaving") and r["rationale"][0].startswith("R1")
    assert r["predicted"]["feasible"]
    big = sim_run("plan", scen((13, 13, 13, 13), [], nodes=4))
    assert big["rationale"][0].startswith("R2")


def test_search_dominates_recommend_on_a_small_box():
    """Planner oracle property: exhaustive_search >= recommend."""
    s = scen((1.3, 0.35, 1.3, 0.35), [], per=2)
    rec = sim_run("plan", s)
    opt = sim_run("search", s)
    assert opt["candidates_feasible"] >= 1
    assert opt["predicted"]["throughput_samples_per_sec"] >= rec["predicted"]["throughput_samples_per_sec"] * (1 - 1e-9)


def test_collective_time_examples_through_disaggregated_paramsync():
    """ParamSync is a Broadcast of 2 P bytes: its simulated comm event lasts
    alpha + 2P / B on the synced devices."""
    s = scen((1, 1, 1, 1), [{"name": "disaggregated", "zero_level": 0, "tp_gen": 1, "batch": 8}],
             cost_model={"alpha_us": 0})
    tr = sim_run("trace", s)
    ps = [e for e in tr["traceEvents"] if e["ph"] == "X" and e["cat"] == "Collective" and e["name"].startswith("sync:")]
    assert ps
    assert abs(ps[0]["dur"] * 1e-6 - 2e9 / 600e9) < 1e-6


def test_cli_exit_codes(tmp_path):
    from paper_2312_11819_b200 import cli
    good = tmp_path / "s.json"
    good.write_text(json.dumps(scen((7, 7, 7, 7), [{"name": "colocated", "zero_level": 3, "batch": 8}])))
    out = tmp_path / "trace.json"
    assert cli.main(["trace", "--config", str(good), "--out", str(out)]) == 0
    assert json.loads(out.read_text())["traceEvents"]
    assert cli.main(["compare", "--config", str(good), "--format", "csv"]) == 0
    bad = tmp_path / "b.json"
    bad.write_text(json.dumps(scen((65, 65, 65, 65), [{"name": "colocated", "zero_level": 3, "batch": 8}])))
    assert cli.main(["simulate", "--config", str(bad)]) == 3
    bad.write_text('{"workload": {"batch": 4, "typo": 1}}')
    assert cli.main(["simulate", "--config", str(bad)]) == 2


def test_b200_scenario_file_runs():
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(__file__)), "scenarios", "c3_8xb200.json")
    rows = sim_run("compare", open(path).read())["rows"]
    assert {r["name"] for r in rows} == {"colocated", "interleaving1", "interleaving2", "disaggregated"}
