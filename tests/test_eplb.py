"""EPLB comparator restatement (paper_2604_19503_b200/eplb.py) vs the imported
reference (moesim/balancers.py:51-199, costmodel.py:96-112): fuzzed on random
loads, budgets, window sizes and cluster shapes, and chained rebalances."""

import numpy as np
import pytest

from paper_2604_19503_b200 import eplb
from paper_2604_19503_b200.policy import ClusterConfig, ExpertPlacement, place_experts_static


def _ref_cfg(reference, cfg):
    return reference.ClusterConfig(num_ranks=cfg.num_ranks, num_layers=cfg.num_layers,
                                   experts_per_rank=cfg.experts_per_rank, bytes_per_expert=cfg.bytes_per_expert)


def test_state_validation(reference):
    from moesim.balancers import EplbState as RefState

    for kw in ({"window_size": 0}, {"interval": 0}, {"redundant_budget": -1}):
        with pytest.raises(ValueError):
            RefState(**kw)
        with pytest.raises(ValueError):
            eplb.EplbState(**kw)
    with pytest.raises(ValueError):
        eplb.eplb_predicted_loads(eplb.EplbState())
    with pytest.raises(ValueError):
        eplb.eplb_observe(eplb.EplbState(), np.ones(3), 4)


@pytest.mark.parametrize("seed", range(40))
def test_rebalance_matches_reference(reference, seed):
    from moesim import balancers as rb

    rng = np.random.default_rng(seed)
    R = int(rng.choice([2, 4, 8]))
    epr = int(rng.choice([1, 2, 4, 8, 16]))
    cfg = ClusterConfig(R, int(rng.integers(1, 5)), epr, 1 << 20)
    rcfg = _ref_cfg(reference, cfg)
    E = R * epr
    kw = dict(window_size=int(rng.integers(1, 6)), interval=int(rng.integers(1, 4)),
              redundant_budget=int(rng.integers(0, 2 * E)))
    ours, ref = eplb.EplbState(**kw), rb.EplbState(**kw)
    place, rplace = place_experts_static(cfg), reference.place_experts_static(rcfg)
    for step in range(6):
        loads = rng.integers(0, 50, E).astype(np.float64)
        if rng.random() < 0.3:
            loads[:] = loads[0]  # ties everywhere
        eplb.eplb_observe(ours, loads, E)
        rb.eplb_observe(ref, loads, E)
        np.testing.assert_array_equal(eplb.eplb_predicted_loads(ours), rb.eplb_predicted_loads(ref))
        if ref.iterations_since_rebalance < ref.interval:
            with pytest.raises(ValueError):
                eplb.eplb_rebalance(ours, cfg, place)
            continue
        place, moved = eplb.eplb_rebalance(ours, cfg, place)
        rplace, rmoved = rb.eplb_rebalance(ref, rcfg, rplace)
        assert place.assignment == rplace.assignment
        assert place.redundant_count == rplace.redundant_count and moved == rmoved
        assert ours.iterations_since_rebalance == ref.iterations_since_rebalance == 0
        from moesim.costmodel import memory_overhead

        assert eplb.memory_overhead(cfg, place) == memory_overhead(rcfg, rplace)


def test_rank_rows_match_aggregate(reference):
    rng = np.random.default_rng(7)
    cfg = ClusterConfig(4, 1, 4, 1)
    st = eplb.EplbState(window_size=1, interval=1, redundant_budget=5)
    eplb.eplb_observe(st, rng.integers(0, 100, 16).astype(float), 16)
    place, _ = eplb.eplb_rebalance(st, cfg, place_experts_static(cfg))
    pairs = rng.integers(0, 1000, 16)
    rows = eplb.rank_expert_rows(pairs, place, 4)
    assert (rows.sum(0) == pairs).all()
    rplace = reference.ExpertPlacement(assignment=place.assignment, redundant_count=place.redundant_count)
    loads = reference.aggregate_rank_loads({e: (int(p), 0) for e, p in enumerate(pairs)}, rplace, 4)
    assert [l.total for l in loads] == rows.sum(1).tolist()


@pytest.mark.parametrize("kw", [dict(window_size=1, interval=1, redundant_budget=8),
                                dict(window_size=2, interval=2, redundant_budget=3)])
def test_schedule_matches_reference_run(reference, golden, kw):
    """Rebalance iterations, replicas moved and the max replica count equal the
    reference simulator's on its own trace (engine.py:170-255)."""
    import json

    from moesim import balancers as rb
    from moesim import engine as reng
    from moesim import tracegen as rtg
    from moesim.costmodel import CostParams
    from paper_2604_19503_b200.replay import read_trace

    meta = json.loads((golden / "trace_plans.json").read_text())
    cfg = ClusterConfig(**meta["cluster"])
    trace = read_trace(golden / "trace_ref_default.csv", cfg)
    sched = eplb.eplb_schedule(trace, eplb.EplbState(**kw))
    rtrace = rtg.read_trace(golden / "trace_ref_default.csv", _ref_cfg(reference, cfg))
    rrun = reng.simulate_run(rtrace, "eplb", CostParams(), eplb_state=rb.EplbState(**kw))
    ours = [(it, m) for it, (_, m) in enumerate(sched) if m is not None]
    assert ours == [(e.iteration, e.replicas_moved) for e in rrun.migration_events]
    assert max(p.redundant_count for p, _ in sched) == rrun.max_redundant_count


def test_memory_overhead_rounding_matches_reference(reference):
    """Odd bytes_per_expert and non-power-of-two rank counts: the half-to-even
    rounding must see the reference's operation order (costmodel.py:105-111)."""
    from moesim.costmodel import memory_overhead

    rng = np.random.default_rng(11)
    cases = [(1, 7, 10, 45, 0)] + [
        (int(rng.integers(1, 6)), int(rng.integers(1, 4000)), int(rng.integers(1, 13)),
         int(rng.integers(1, 9)), int(rng.integers(0, 20))) for _ in range(3000)]
    for L, bpe, R, epr, red in cases:
        cfg = ClusterConfig(R, L, epr, bpe)
        E = R * epr
        hosts = [(e // epr,) for e in range(E)]
        for j in range(red):  # replicas on other ranks
            e = j % E
            extra = (hosts[e][-1] + 1) % R
            if extra not in hosts[e]:
                hosts[e] = hosts[e] + (extra,)
        red_n = sum(len(h) - 1 for h in hosts)
        place = ExpertPlacement(tuple(hosts), red_n)
        rplace = reference.ExpertPlacement(assignment=tuple(hosts), redundant_count=red_n)
        assert eplb.memory_overhead(cfg, place) == memory_overhead(_ref_cfg(reference, cfg), rplace), \
            (L, bpe, R, epr, red_n)
