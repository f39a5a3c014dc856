"""Trace replay on the B200: the reference generator's prefill-scale EP8 trace
(tests/golden/trace_prefill_ep8.csv) is executed layer by layer through the
real router -> device plan -> dispatch -> GEMMs -> combine on the Kimi-VL shape
(64 experts = the trace's 8 ranks x 8 experts). The router must pick exactly
the replayed experts, the device counts must equal the replay's, and the
device plan must equal the reference's plan on the same trace records
(tests/golden/trace_plans.json)."""

import json

import numpy as np
import pytest
import torch

from paper_2604_19503_b200.policy import ClusterConfig
from paper_2604_19503_b200.replay import TraceReplay, read_trace, speedup_report, write_run

pytestmark = pytest.mark.gpu


def test_prefill_trace_replay_parity_and_bridge(golden, tmp_path):
    meta = json.loads((golden / "trace_plans.json").read_text())
    cluster = ClusterConfig(**meta["cluster"])
    trace = read_trace(golden / "trace_prefill_ep8.csv", cluster)
    rep = TraceReplay(torch, "kimi", trace)
    runs, checks = rep.run(iterations=[0])
    assert len(checks) == 4 * 3
    for c in checks:
        assert c["routing_equal"] and c["counts_equal"], c
        assert c["plan_equal_pairs"] and c["plan_equal_trace"], c
    ref = meta["trace_prefill_ep8.csv"]
    for (it, la), plan in runs["realb"].plans.items():
        assert [p.value for p in plan.per_rank_precision] == ref[f"{it},{la}"]["realb"]["precisions"]
    summaries = {s: write_run(r, trace, tmp_path / s, "t") for s, r in runs.items()}
    rows = {r["strategy"]: r for r in speedup_report(summaries)}
    # every layer of this trace activates ReaLB on the vision-hot rank
    assert all(p.active for p in runs["realb"].plans.values())
    assert rows["realb"]["layer_speedup"] > 1.2
    assert rows["fp4all"]["layer_speedup"] >= rows["realb"]["layer_speedup"] * 0.9
    for s in ("baseline", "realb", "fp4all"):
        assert (tmp_path / s / "layers.csv").exists() and (tmp_path / s / "summary.json").exists()


def test_eplb_comparator_runs_on_gpu(golden, tmp_path):
    """EPLB (the reference's replication balancer, one-iteration window) next to
    ReaLB on the prefill trace: placements with replicas are timed on the GPU,
    migrations charged, and the run files written in the reference schema."""
    meta = json.loads((golden / "trace_plans.json").read_text())
    cluster = ClusterConfig(**meta["cluster"])
    trace = read_trace(golden / "trace_prefill_ep8.csv", cluster)
    rep = TraceReplay(torch, "kimi", trace)
    runs, _ = rep.run(strategies=("baseline", "realb", "eplb", "async-eplb"), check=False,
                      eplb_state=dict(window_size=1, interval=1, redundant_budget=8))
    ev = runs["eplb"].migration_events
    assert [e.iteration for e in ev] == [1] and ev[0].replicas_moved > 0
    assert runs["async-eplb"].migration_events[0].charged_ns <= ev[0].charged_ns
    assert runs["eplb"].max_redundant_count == 8
    summaries = {s: write_run(r, trace, tmp_path / s, "t") for s, r in runs.items()}
    rows = {r["strategy"]: r for r in speedup_report(summaries)}
    assert summaries["eplb"]["mem_delta_bytes"] > 0 and rows["eplb"]["text_exposure"] == 0.0
    # after its rebalance EPLB evens the ranks out: iteration 1 compute-only beats baseline
    it1 = lambda s: sum(t.compute_only_ns for (i, _), t in runs[s].layer_timings.items() if i == 1)
    assert it1("eplb") < it1("baseline")
