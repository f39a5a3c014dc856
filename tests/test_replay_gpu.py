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
