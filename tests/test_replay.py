"""Trace replay + measured-timing bridge, host side.

Fixtures: tests/golden/trace_*.csv and trace_plans.json were written by the
reference's own generator, writer and policy (tests/golden/make_trace.py)."""

import argparse
import json

import numpy as np
import pytest

from paper_2604_19503_b200.moe import LayerTiming, PipelineMode, RankPhases
from paper_2604_19503_b200.policy import (ClusterConfig, RealbParams, aggregate_rank_loads,
                                          place_experts_static, plan_for)
from paper_2604_19503_b200.replay import (MeasuredRun, TraceMismatchError, TraceParseError, pair_loads,
                                          read_trace, replay_pair_counts, routing_from_expert_loads,
                                          speedup_report, write_run, write_trace)

TRACES = ("trace_ref_default.csv", "trace_prefill_ep8.csv")


@pytest.fixture(scope="module")
def cluster(golden):
    return ClusterConfig(**json.loads((golden / "trace_plans.json").read_text())["cluster"])


def _plan_record(plan):
    return {"precisions": [p.value for p in plan.per_rank_precision], "hot": sorted(plan.hot_ranks),
            "vision": sorted(plan.vision_heavy_ranks), "active": plan.active}


@pytest.mark.parametrize("name", TRACES)
def test_trace_round_trip_bytes(golden, cluster, tmp_path, name):
    tr = read_trace(golden / name, cluster)
    write_trace(tr, tmp_path / name)
    assert (tmp_path / name).read_bytes() == (golden / name).read_bytes()


def test_trace_errors(golden, cluster, tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("iter,layer,expert,v,t\n0,0,0,1,1\n")
    with pytest.raises(TraceParseError):
        read_trace(p, cluster)
    p.write_text("iter,layer,expert,vision_tokens,text_tokens\n0,0,0,1\n")
    with pytest.raises(TraceParseError):
        read_trace(p, cluster)
    p.write_text("iter,layer,expert,vision_tokens,text_tokens\n0,0,99,1,1\n")
    with pytest.raises(TraceMismatchError):
        read_trace(p, cluster)
    p.write_text("iter,layer,expert,vision_tokens,text_tokens\n0,0,1,1,1\n0,0,1,2,2\n")
    with pytest.raises(TraceMismatchError):
        read_trace(p, cluster)


@pytest.mark.parametrize("name", TRACES)
def test_host_plans_match_reference(golden, cluster, name):
    """Our policy on the trace = the reference's plans (fixture), and on the
    replay's k x pair loads with the k-scaled gate it is the same plan (D2)."""
    ref = json.loads((golden / "trace_plans.json").read_text())[name]
    tr = read_trace(golden / name, cluster)
    pl = place_experts_static(cluster)
    k = 6
    pk = RealbParams(global_batch_threshold=2048 * k)
    for key, per in ref.items():
        it, la = map(int, key.split(","))
        loads = tr.layer_loads(it, la)
        for s, want in per.items():
            assert _plan_record(plan_for(s, aggregate_rank_loads(loads, pl, 8), cluster, RealbParams())) == want
            assert _plan_record(plan_for(s, aggregate_rank_loads(pair_loads(loads, k), pl, 8), cluster, pk)) == want


@pytest.mark.parametrize("name", TRACES)
def test_routing_reproduces_rank_loads(golden, cluster, name):
    tr = read_trace(golden / name, cluster)
    k, E, epr = 6, 64, 8
    for it in range(tr.num_iterations):
        for la in range(cluster.num_layers):
            loads = tr.layer_loads(it, la)
            mod, idx = routing_from_expert_loads(loads, E, k, epr, seed=it * 7 + la)
            assert len(mod) == sum(v + t for v, t in loads.values())
            s = np.sort(idx, axis=1)
            assert (s[:, 1:] != s[:, :-1]).all(), "k distinct experts per token"
            got = replay_pair_counts(mod, idx, E)
            want = np.zeros((E, 2), np.int64)
            for e, vt in loads.items():
                want[e] = (k * vt[0], k * vt[1])
            assert (got.reshape(8, epr, 2).sum(1) == want.reshape(8, epr, 2).sum(1)).all()
            # experts under the top-k cap keep their exact k x counts
            n = np.array([want[:, 0].sum() // k, want[:, 1].sum() // k])
            if (want <= n).all():
                assert (got == want).all()


def test_routing_cap_without_ranks_raises():
    with pytest.raises(ValueError):
        routing_from_expert_loads({0: (10, 0), 1: (1, 0)}, 4, 2)
    mod, idx = routing_from_expert_loads({0: (3, 1), 1: (3, 1), 2: (2, 2), 3: (0, 0)}, 4, 2)
    assert (replay_pair_counts(mod, idx, 4) == [[6, 2], [6, 2], [4, 4], [0, 0]]).all()


def _fake_run(strategy, cluster, trace, scale):
    run = MeasuredRun(strategy, timing_source="test")
    pl = place_experts_static(cluster)
    for it in range(trace.num_iterations):
        for la in range(cluster.num_layers):
            R = cluster.num_ranks
            loads = aggregate_rank_loads(trace.layer_loads(it, la), pl, R)
            plan = plan_for(strategy, loads, cluster, RealbParams())
            phases = tuple(RankPhases(1000, 50 * r * (strategy != "baseline"), 2000 + r, int(scale * (3000 + 10 * r)),
                                      2000) for r in range(R))
            mode = PipelineMode.OVERLAPPED if strategy != "baseline" and plan.active else PipelineMode.SEQUENTIAL
            totals = tuple(p.total(mode, plan.per_rank_precision[r].value == "w4a4") for r, p in enumerate(phases))
            lat = max(totals)
            run.layer_timings[(it, la)] = LayerTiming(phases, totals, lat, max(p.compute_ns for p in phases),
                                                      totals.index(lat), mode)
            run.plans[(it, la)] = plan
    return run


def test_bridge_files_match_reference_writers(golden, cluster, tmp_path, reference):
    """layers.csv / ranks.csv / events.csv are byte-identical to the reference's
    writers (engine.py:258-288) on the same timings, and summary.json carries
    summarize_run's fields with the reference's text_exposure (metrics.py:72-90)."""
    from moesim import engine as reng
    from moesim import metrics as rmet
    from moesim import tracegen as rtg
    from moesim.core import ClusterConfig as RCluster

    name = "trace_ref_default.csv"
    run = _fake_run("realb", cluster, read_trace(golden / name, cluster), 0.5)
    meta = write_run(run, read_trace(golden / name, cluster), tmp_path / "ours", "abc", ranks_iters=(0, 1))
    rcfg = RCluster(**json.loads((golden / "trace_plans.json").read_text())["cluster"])
    rtrace = rtg.read_trace(golden / name, rcfg)
    rres = reng.RunResult(strategy="realb")
    for key, t in run.layer_timings.items():
        rres.layer_timings[key] = reng.LayerTiming(
            tuple(reng.RankPhases(p.schedule_ns, p.transform_ns, p.dispatch_ns, p.compute_ns, p.combine_ns)
                  for p in t.per_rank), t.per_rank_total_ns, t.layer_latency_ns, t.compute_only_ns,
            t.critical_rank, reng.PipelineMode(t.pipeline_mode.value))
        rloads = reference.aggregate_rank_loads(rtrace.layer_loads(*key), reference.place_experts_static(rcfg), 8)
        rres.plans[key] = reference.plan_for("realb", rloads, rcfg)
    reng.write_layers_csv(rres, tmp_path / "layers.csv")
    reng.write_ranks_csv(rres, [0, 1], tmp_path / "ranks.csv")
    reng.write_events_csv(rres, tmp_path / "events.csv")
    for f in ("layers.csv", "ranks.csv", "events.csv"):
        assert (tmp_path / "ours" / f).read_bytes() == (tmp_path / f).read_bytes(), f
    summ = rmet.summarize_run(rres, rtrace, rcfg)
    assert meta["e2e_time_ns"] == summ.e2e_time_ns
    assert meta["compute_only_total_ns"] == summ.compute_only_total_ns
    assert meta["text_exposure"] == summ.text_exposure


def test_reference_compare_reads_our_runs(golden, cluster, tmp_path, reference):
    """The unmodified ``moesim compare`` (cli.py:157-185) consumes our run
    directories; its report equals ours (metrics.speedup_report)."""
    from moesim import cli as rcli

    tr = read_trace(golden / "trace_ref_default.csv", cluster)
    metas = {}
    for s, scale in (("baseline", 1.0), ("realb", 0.6), ("fp4all", 0.4)):
        metas[s] = write_run(_fake_run(s, cluster, tr, scale), tr, tmp_path / s, "same-trace")
    out = tmp_path / "report.csv"
    rc = rcli.cmd_compare(argparse.Namespace(runs=[str(tmp_path / s) for s in metas], out=str(out)))
    assert rc == 0
    rows = out.read_text().splitlines()
    ours = speedup_report(metas)
    assert rows[0] == "strategy,layer_speedup,e2e_speedup,mem_delta_bytes,migration_bytes,text_exposure"
    for line, r in zip(rows[1:], ours):
        f = line.split(",")
        assert f[0] == r["strategy"]
        assert float(f[1]) == pytest.approx(r["layer_speedup"], rel=1e-5)
        assert float(f[2]) == pytest.approx(r["e2e_speedup"], rel=1e-5)
        assert float(f[5]) == pytest.approx(r["text_exposure"], rel=1e-5, abs=1e-12)
    realb = next(r for r in ours if r["strategy"] == "realb")
    assert realb["layer_speedup"] > 1.0
