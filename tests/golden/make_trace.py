"""Generate the committed routing-trace fixtures by running the REFERENCE's own
trace generator (moesim/tracegen.py:141-185, write_trace :255-260) and its
policy on them, for the trace-replay parity tests (tests/test_replay*.py).

Run in the build container (where /root/reference exists):
    python tests/golden/make_trace.py

* trace_ref_default.csv — the reference test suite's calibrated cluster
  (8 ranks x 8 experts, 4 layers; pkg/tests/conftest.py:17-30) and spec
  (seed 2024, defaults: 4096 tokens/iteration), first 3 iterations.
* trace_prefill_ep8.csv — the same generator at prefill scale (65536 tokens
  per iteration = 8192 per EP8 rank, the bench workload), 2 iterations x 4 layers.
* trace_plans.json — the reference's per-(iteration, layer) realb / fp4all plans
  on both traces (aggregate_rank_loads + plan_for, engine.py:205-208).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from moesim import (  # noqa: E402
    ClusterConfig,
    RealbParams,
    TraceSpec,
    aggregate_rank_loads,
    generate_trace,
    place_experts_static,
    plan_for,
)
from moesim.tracegen import write_trace  # noqa: E402

CLUSTER = dict(num_ranks=8, num_layers=4, experts_per_rank=8, bytes_per_expert=4 * 1024 * 1024)
TRACES = {
    "trace_ref_default.csv": TraceSpec(num_iterations=3, seed=2024),
    "trace_prefill_ep8.csv": TraceSpec(num_iterations=2, seed=2024, tokens_per_iteration_mean=65536,
                                       tokens_per_iteration_jitter=2048),
}


def plan_record(plan):
    return {"precisions": [p.value for p in plan.per_rank_precision], "hot": sorted(plan.hot_ranks),
            "vision": sorted(plan.vision_heavy_ranks), "active": plan.active}


def main():
    cfg = ClusterConfig(**CLUSTER)
    placement = place_experts_static(cfg)
    plans = {"cluster": CLUSTER}
    for name, spec in TRACES.items():
        trace = generate_trace(cfg, spec)
        write_trace(trace, HERE / name)
        per = {}
        for it in range(trace.num_iterations):
            for la in range(cfg.num_layers):
                loads = aggregate_rank_loads(trace.layer_loads(it, la), placement, cfg.num_ranks)
                per[f"{it},{la}"] = {s: plan_record(plan_for(s, loads, cfg, RealbParams()))
                                     for s in ("baseline", "fp4all", "realb")}
        plans[name] = per
    (HERE / "trace_plans.json").write_text(json.dumps(plans, indent=1, sort_keys=True) + "\n")
    print("wrote", ", ".join(TRACES), "trace_plans.json")


if __name__ == "__main__":
    main()
