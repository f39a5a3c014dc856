"""CPU ORACLE of the ReaLB precision policy — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Plain-Python restatement of the reference's per-rank load aggregation and
policy, with the reference's integer sums and fp64 operation order, so the
CPU arms of bench.py can run the whole path without the product library:

  aggregate_rank_loads   moesim/core.py:106-130 (+ _split_evenly :100-103)
  plan_realb             moesim/balancers.py:89-122
  plan_baseline          moesim/balancers.py:66-74
  plan_fp4_all           moesim/balancers.py:77-86

Loads are (rank, vision, text) tuples; a plan is a dict {"precision": [0/1 per
rank id], "hot": frozenset, "vision": frozenset, "active": bool} (1 = W4A4).
Pinned by tests/test_oracle.py against tests/golden/policy_cases.json (400
reference outputs) and a live fuzz against the imported reference.
"""

from __future__ import annotations


def _split(count: int, parts: int) -> list[int]:
    base, rem = divmod(count, parts)
    return [base + (i < rem) for i in range(parts)]


def aggregate_rank_loads(expert_loads: dict, assignment, num_ranks: int) -> list[tuple[int, int, int]]:
    """expert -> (v, t) counts summed onto the hosting ranks of ``assignment``
    (expert -> tuple of hosts); replicas split with the remainder on the lowest
    rank ids. Unknown experts raise ValueError (PlacementMismatchError upstream)."""
    vis, txt = [0] * num_ranks, [0] * num_ranks
    for e, (v, t) in expert_loads.items():
        if not 0 <= e < len(assignment):
            raise ValueError(f"expert {e} not in placement")
        hosts = sorted(set(assignment[e]))
        for h, sv, st in zip(hosts, _split(v, len(hosts)), _split(t, len(hosts))):
            vis[h] += sv
            txt[h] += st
    return [(r, vis[r], txt[r]) for r in range(num_ranks)]


def plan_baseline(loads):
    return {"precision": [0] * len(loads), "hot": frozenset(), "vision": frozenset(), "active": False}


def plan_fp4_all(loads):
    every = frozenset(range(len(loads)))
    return {"precision": [1] * len(loads), "hot": every, "vision": every, "active": True}


def plan_realb(loads, C: float = 1.0, Md: float = 0.7, threshold: int = 2048, isolated: bool = False):
    """W4A4 on ranks both hot (total / (sum / R) > C) and vision-heavy
    (v / total > Md; any loaded rank when modality-isolated), gated on the
    global sum; sets are rank ids and precision is indexed by rank id."""
    total = sum(v + t for _, v, t in loads)
    if total < threshold or total == 0:
        return plan_baseline(loads)
    ideal = total / len(loads)
    hot = frozenset(r for r, v, t in loads if (v + t) / ideal > C)
    if isolated:
        vision = frozenset(r for r, v, t in loads if v + t > 0)
    else:
        vision = frozenset(r for r, v, t in loads if v + t > 0 and v / (v + t) > Md)
    acc = hot & vision
    return {"precision": [1 if r in acc else 0 for r in range(len(loads))], "hot": hot, "vision": vision,
            "active": True}


def plan_for(strategy: str, loads, C=1.0, Md=0.7, threshold=2048, isolated=False):
    if strategy == "fp4all":
        return plan_fp4_all(loads)
    if strategy in ("realb", "realb-seq"):
        return plan_realb(loads, C, Md, threshold, isolated)
    return plan_baseline(loads)
