"""C-ABI library: loads without a GPU, exports every symbol include/realb.h
declares, and its host policy (realb_plan) reproduces moesim.plan_realb."""

import json
import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.policy import (
    ClusterConfig, ExpertPlacement, PlacementMismatchError, Precision, RankLoad, RealbParams,
    aggregate_rank_loads, place_experts_static, plan_baseline, plan_for, plan_fp4_all, plan_realb,
    rank_loads_from_counts)


def header_symbols():
    from pathlib import Path

    text = (Path(__file__).resolve().parents[1] / "include" / "realb.h").read_text()
    return sorted(set(re.findall(r"REALB_API\s+[\w\s\*]+?\b(realb_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with realb.h"
    assert lib.realb_abi_version() == 1


def test_error_reporting_without_gpu():
    with pytest.raises(_lib.RealbError, match="RealbParams"):
        vt = np.zeros((2, 2), np.int64)
        prec = np.zeros(2, np.uint8)
        _lib.call("realb_plan", vt.ctypes.data, 2, -1.0, 0.7, 0, 0, prec.ctypes.data, None)


def _cfg(R, iso=False, epr=1):
    return ClusterConfig(num_ranks=R, num_layers=1, experts_per_rank=epr, bytes_per_expert=1,
                         modality_isolated=iso)


def test_policy_matches_reference_fixture(golden):
    cases = json.loads((golden / "policy_cases.json").read_text())
    for cs in cases:
        R = len(cs["v"])
        loads = [RankLoad(r, cs["v"][r], cs["t"][r]) for r in range(R)]
        plan = plan_realb(loads, RealbParams(cs["C"], cs["Md"], cs["thr"]), _cfg(R, cs["iso"]))
        e = cs["expect"]
        assert [p.value for p in plan.per_rank_precision] == e["prec"], cs
        assert sorted(plan.hot_ranks) == e["hot"], cs
        assert sorted(plan.vision_heavy_ranks) == e["vision"], cs
        assert plan.active == e["active"], cs


# reference unit cases, tests/test_balancers.py:64-108
def _mk(totals, fracs=None):
    out = []
    for r, t in enumerate(totals):
        f = 1.0 if fracs is None else fracs[r]
        v = int(round(t * f))
        out.append(RankLoad(r, v, t - v))
    return out


def test_reference_unit_cases():
    p = plan_realb(_mk([1000, 1000, 100, 100], [0.9, 0.5, 0.5, 0.5]), RealbParams(global_batch_threshold=0), _cfg(4))
    assert p.hot_ranks == {0, 1} and 0 in p.vision_heavy_ranks and 1 not in p.vision_heavy_ranks
    assert p.per_rank_precision[:2] == (Precision.W4A4, Precision.W16A16)
    assert plan_realb(_mk([100] * 8), RealbParams(global_batch_threshold=0), _cfg(8)).hot_ranks == frozenset()
    loads = _mk([100] * 8)
    assert plan_realb(loads, RealbParams(), _cfg(8)) == plan_baseline(loads)
    assert not plan_realb(_mk([0] * 8), RealbParams(global_batch_threshold=0), _cfg(8)).active
    iso = plan_realb(_mk([1000] + [100] * 7, [0.0] * 8), RealbParams(global_batch_threshold=0), _cfg(8, True))
    assert iso.per_rank_precision[0] is Precision.W4A4
    with pytest.raises(ValueError):
        plan_realb(_mk([1, 2]), RealbParams(), _cfg(3))
    # one GPU: never hot (balancers.py:103-104)
    assert plan_realb(_mk([10**6]), RealbParams(), _cfg(1)).accelerated_ranks == frozenset()


def test_plan_for_and_fixed_plans():
    loads = _mk([5000] + [100] * 7)
    for tag in ("baseline", "eplb", "async-eplb"):
        assert plan_for(tag, loads, _cfg(8)) == plan_baseline(loads)
    assert plan_for("fp4all", loads, _cfg(8)) == plan_fp4_all(loads)
    prm = RealbParams(global_batch_threshold=0)
    assert plan_for("realb-seq", loads, _cfg(8), prm) == plan_for("realb", loads, _cfg(8), prm)
    with pytest.raises(ValueError, match="unknown strategy"):
        plan_for("nope", _mk([1]), _cfg(1))


@given(totals=st.lists(st.integers(0, 10_000), min_size=8, max_size=8),
       fracs=st.lists(st.floats(0.0, 1.0), min_size=8, max_size=8),
       C=st.floats(0.25, 3.0), Md=st.floats(0.0, 1.0), thr=st.integers(0, 40_000),
       iso=st.booleans())
@settings(max_examples=300, deadline=None)
def test_policy_fuzz_against_live_reference(reference, totals, fracs, C, Md, thr, iso):
    from moesim import ClusterConfig as RC, RankLoad as RL, RealbParams as RP, plan_realb as rplan

    loads = _mk(totals, fracs)
    ref = rplan([RL(l.rank, l.vision_tokens, l.text_tokens) for l in loads], RP(C, Md, thr),
                RC(8, 1, 1, 1, iso))
    got = plan_realb(loads, RealbParams(C, Md, thr), _cfg(8, iso))
    assert [p.value for p in got.per_rank_precision] == [p.value for p in ref.per_rank_precision]
    assert got.hot_ranks == ref.hot_ranks and got.vision_heavy_ranks == ref.vision_heavy_ranks
    assert got.active == ref.active


@given(totals=st.lists(st.integers(0, 10_000), min_size=4, max_size=4),
       fracs=st.lists(st.floats(0.0, 1.0), min_size=4, max_size=4),
       perm=st.permutations(range(4)), dup=st.booleans(), iso=st.booleans())
@settings(max_examples=200, deadline=None)
def test_policy_rank_ids_not_positions(reference, totals, fracs, perm, dup, iso):
    """Loads out of rank order (and duplicate rank ids): the hot / vision sets are
    rank ids and precision is indexed by rank id (balancers.py:104-118)."""
    from moesim import ClusterConfig as RC, RankLoad as RL, RealbParams as RP, plan_realb as rplan

    base = _mk(totals, fracs)
    ranks = list(perm)
    if dup:
        ranks[1] = ranks[0]
    loads = [RankLoad(r, l.vision_tokens, l.text_tokens) for r, l in zip(ranks, base)]
    ref = rplan([RL(l.rank, l.vision_tokens, l.text_tokens) for l in loads], RP(1.0, 0.7, 0),
                RC(4, 1, 1, 1, iso))
    got = plan_realb(loads, RealbParams(1.0, 0.7, 0), _cfg(4, iso))
    assert [p.value for p in got.per_rank_precision] == [p.value for p in ref.per_rank_precision]
    assert got.hot_ranks == ref.hot_ranks and got.vision_heavy_ranks == ref.vision_heavy_ranks
    assert got.active == ref.active


def test_policy_advisor_case(reference):
    from moesim import ClusterConfig as RC, RankLoad as RL, RealbParams as RP, plan_realb as rplan

    raw = [(1, 900, 100), (0, 10, 10), (2, 10, 10)]
    ref = rplan([RL(*t) for t in raw], RP(1.0, 0.7, 0), RC(3, 1, 1, 1))
    got = plan_realb([RankLoad(*t) for t in raw], RealbParams(1.0, 0.7, 0), _cfg(3))
    assert [p.value for p in got.per_rank_precision] == [p.value for p in ref.per_rank_precision]
    assert got.per_rank_precision[1] is Precision.W4A4


def test_aggregation_matches_reference(reference):
    import random

    from moesim import ExpertPlacement as RP, aggregate_rank_loads as ragg

    rng = random.Random(11)
    for _ in range(60):
        n_e, n_r = rng.randint(1, 12), rng.randint(1, 5)
        assign = tuple(tuple(sorted(rng.sample(range(n_r), rng.randint(1, n_r)))) for _ in range(n_e))
        red = sum(len(h) - 1 for h in assign)
        el = {e: (rng.randint(0, 100), rng.randint(0, 100)) for e in range(n_e)}
        a = aggregate_rank_loads(el, ExpertPlacement(assign, red), n_r)
        b = ragg(el, RP(assign, red), n_r)
        assert [(x.vision_tokens, x.text_tokens) for x in a] == [(x.vision_tokens, x.text_tokens) for x in b]
    with pytest.raises(PlacementMismatchError):
        aggregate_rank_loads({5: (1, 1)}, ExpertPlacement(((0,),)), 1)


def test_static_placement_and_count_fast_path():
    cfg = _cfg(4, epr=3)
    pl = place_experts_static(cfg)
    assert pl.assignment[0] == (0,) and pl.assignment[11] == (3,)
    rng = np.random.default_rng(0)
    vt = rng.integers(0, 50, (12, 2))
    fast = rank_loads_from_counts(vt, cfg)
    slow = aggregate_rank_loads({e: tuple(map(int, vt[e])) for e in range(12)}, pl, 4)
    assert fast == slow
    plan = plan_realb(fast, RealbParams(global_batch_threshold=0), cfg)
    ep = plan.expert_precision(pl)
    for e in range(12):
        assert ep[e] == plan.per_rank_precision[e // 3].code
