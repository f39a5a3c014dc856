"""EPLB comparator: the reference's expert-replication load
balancer, restated so its placements can be executed and timed on the B200 next
to ReaLB.

  EplbState              moesim/balancers.py:51-63
  eplb_observe           moesim/balancers.py:125-135
  eplb_predicted_loads   moesim/balancers.py:138-141
  eplb_rebalance         moesim/balancers.py:143-199   (replicate the predicted-hottest
                         experts, then longest-processing-time packing onto ranks)
  memory_overhead        moesim/costmodel.py:96-112
  migration bytes        moesim/costmodel.py:87-93 (the latency is measured-bandwidth
                         based here: bytes / NVLink peer bandwidth)

Same names, arguments, results and errors as the reference; `tests/test_eplb.py`
fuzzes every function against the imported reference.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .policy import ClusterConfig, ExpertPlacement


@dataclass
class EplbState:
    window_size: int = 100
    interval: int = 100
    redundant_budget: int = 8
    window: deque = field(default_factory=deque)
    iterations_since_rebalance: int = 0

    def __post_init__(self):
        if self.window_size < 1 or self.interval < 1:
            raise ValueError("window_size and interval must be >= 1")
        if self.redundant_budget < 0:
            raise ValueError("redundant_budget must be >= 0")


def eplb_observe(state: EplbState, expert_loads: np.ndarray, num_experts: int) -> None:
    """Push one iteration's per-expert loads into the sliding window."""
    if len(expert_loads) != num_experts:
        raise ValueError(f"expected {num_experts} expert loads, got {len(expert_loads)}")
    state.window.append(np.array(expert_loads, dtype=np.float64))
    while len(state.window) > state.window_size:
        state.window.popleft()
    state.iterations_since_rebalance += 1


def eplb_predicted_loads(state: EplbState) -> np.ndarray:
    """Window mean per expert."""
    if not state.window:
        raise ValueError("window is empty")
    return np.stack(list(state.window)).mean(axis=0)


def eplb_rebalance(state: EplbState, config: ClusterConfig,
                   old_placement: ExpertPlacement) -> tuple[ExpertPlacement, int]:
    """New placement and the number of replicas that land on a rank that did not
    host that expert before. Each of the `redundant_budget` predicted-hottest
    experts (ties to the lowest id) gets one extra replica; the instances, each
    carrying its expert's load / replicas, are packed largest first onto the
    least-loaded rank (ties to the lowest rank) that has a free slot and does not
    host the expert yet (a duplicate host is tolerated only when no such rank
    exists). Slots per rank: experts_per_rank + ceil(budget / num_ranks)."""
    if state.iterations_since_rebalance < state.interval:
        raise ValueError("rebalance called before the interval elapsed")
    pred = eplb_predicted_loads(state)
    E, R = config.total_experts, config.num_ranks
    if len(pred) != E:
        raise ValueError("window dimension does not match config")
    reps = np.ones(E, dtype=np.int64)
    if state.redundant_budget > 0:
        hottest = np.lexsort((np.arange(E), -pred))[: state.redundant_budget]
        reps[hottest] += 1
    slots = config.experts_per_rank + math.ceil(state.redundant_budget / R)
    inst = sorted(((pred[e] / reps[e], e, i) for e in range(E) for i in range(reps[e])),
                  key=lambda t: (-t[0], t[1], t[2]))
    load = [0.0] * R
    used = [0] * R
    hosts: list[list[int]] = [[] for _ in range(E)]
    for share, e, _ in inst:
        cand = [r for r in range(R) if used[r] < slots and r not in hosts[e]] or \
               [r for r in range(R) if used[r] < slots]
        r = min(cand, key=lambda r: (load[r], r))
        load[r] += share
        used[r] += 1
        if r not in hosts[e]:
            hosts[e].append(r)
    assignment = tuple(tuple(sorted(h)) for h in hosts)
    placement = ExpertPlacement(assignment, sum(len(h) - 1 for h in assignment))
    moved = sum(len(set(assignment[e]) - set(old_placement.assignment[e])) for e in range(E))
    state.iterations_since_rebalance = 0
    return placement, moved


def memory_overhead(config: ClusterConfig, placement: ExpertPlacement) -> tuple[int, int]:
    """Per-rank expert weight bytes and the delta over a replica-free placement
    (costmodel.py:96-112; round half to even)."""
    lb = config.num_layers * config.bytes_per_expert  # the reference's operation order
    total = round(lb * (placement.num_experts + placement.redundant_count) / config.num_ranks)
    base = round(lb * placement.num_experts / config.num_ranks)
    return total, total - base


def rank_expert_rows(expert_pairs: np.ndarray, placement: ExpertPlacement, num_ranks: int) -> np.ndarray:
    """[R, E] (token, expert) pairs each rank computes: an expert's pairs split
    evenly over its hosts, remainder to the lowest rank ids — the split
    aggregate_rank_loads uses (core.py:100-130)."""
    E = len(expert_pairs)
    out = np.zeros((num_ranks, E), np.int64)
    for e in range(E):
        hosts = sorted(set(placement.assignment[e]))
        q, rem = divmod(int(expert_pairs[e]), len(hosts))
        for i, h in enumerate(hosts):
            out[h, e] += q + (i < rem)
    return out


def eplb_schedule(trace, state: EplbState, iterations=None) -> list[tuple[ExpertPlacement, int | None]]:
    """The placement each iteration of a trace runs under, and the replicas moved
    by the rebalance at its start (None: no rebalance) — the reference's
    simulate_iteration order (engine.py:181-205, :229-235): rebalance when the
    window is non-empty and the interval has elapsed, then observe the
    iteration's per-expert totals over all layers. Pure function of the trace."""
    from .policy import place_experts_static

    cfg = trace.cluster
    E = cfg.total_experts
    place = place_experts_static(cfg)
    out = []
    for it in (range(trace.num_iterations) if iterations is None else iterations):
        moved = None
        if state.window and state.iterations_since_rebalance >= state.interval:
            place, moved = eplb_rebalance(state, cfg, place)
        out.append((place, moved))
        totals = np.zeros(E, np.int64)
        for la in range(cfg.num_layers):
            for e, (v, t) in trace.layer_loads(it, la).items():
                totals[e] += v + t
        eplb_observe(state, totals, E)
    return out
