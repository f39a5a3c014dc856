"""Host-side EP topology, per-rank load statistics and the ReaLB precision policy.

Drop-in mirror of the reference entry points on the MoE-layer path (same names,
argument meaning and error behaviour):

  Precision, ClusterConfig, ExpertPlacement, RankLoad      moesim/core.py:9-89
  place_experts_static, aggregate_rank_loads               moesim/core.py:92-130
  STRATEGIES, PrecisionPlan, RealbParams                   moesim/balancers.py:19-48
  plan_baseline, plan_fp4_all, plan_realb, plan_for        moesim/balancers.py:66-122, :202-219

``plan_realb`` evaluates the policy in the shipped C library (``realb_plan``,
runtime.cu), whose fp64 operation order is the reference's; the Python layer
only builds the immutable plan record. ``rank_loads_from_counts`` is the fast
path from the router's device-side (vision, text) counts.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from . import _lib

STRATEGIES = ("baseline", "fp4all", "eplb", "async-eplb", "realb", "realb-seq")


class Precision(enum.Enum):
    W16A16 = "w16a16"
    W4A4 = "w4a4"

    @property
    def code(self) -> int:
        return _lib.PREC_W4A4 if self is Precision.W4A4 else _lib.PREC_W16A16


class PlacementMismatchError(ValueError):
    """A load names an expert the placement does not know (core.py:14)."""


@dataclass(frozen=True)
class ClusterConfig:
    num_ranks: int
    num_layers: int
    experts_per_rank: int
    bytes_per_expert: int
    modality_isolated: bool = False

    def __post_init__(self):
        for name, lo in (("num_ranks", 1), ("num_layers", 1), ("experts_per_rank", 1)):
            if getattr(self, name) < lo:
                raise ValueError(f"{name} must be >= {lo}")
        if self.bytes_per_expert <= 0:
            raise ValueError("bytes_per_expert must be > 0")

    @property
    def total_experts(self) -> int:
        return self.num_ranks * self.experts_per_rank


@dataclass(frozen=True)
class ExpertPlacement:
    """expert id -> tuple of hosting ranks (more than one host = a replica)."""

    assignment: tuple[tuple[int, ...], ...]
    redundant_count: int = 0

    def __post_init__(self):
        if any(len(h) == 0 for h in self.assignment):
            bad = next(i for i, h in enumerate(self.assignment) if len(h) == 0)
            raise ValueError(f"expert {bad} has no host")
        implied = sum(len(h) - 1 for h in self.assignment)
        if implied != self.redundant_count:
            raise ValueError(
                f"redundant_count={self.redundant_count} but assignment implies {implied}")

    @property
    def num_experts(self) -> int:
        return len(self.assignment)

    def hosted_experts(self, rank: int) -> list[int]:
        return [e for e, hosts in enumerate(self.assignment) if rank in hosts]

    def hosted_instance_count(self, rank: int) -> int:
        return len(self.hosted_experts(rank))


@dataclass(frozen=True)
class RankLoad:
    """(token, expert) pairs routed to one EP rank, split by modality."""

    rank: int
    vision_tokens: int
    text_tokens: int

    def __post_init__(self):
        if min(self.vision_tokens, self.text_tokens) < 0:
            raise ValueError("token counts must be >= 0")

    @property
    def total(self) -> int:
        return self.vision_tokens + self.text_tokens

    @property
    def vision_ratio(self) -> float:
        t = self.total
        return self.vision_tokens / t if t else 0.0


def place_experts_static(config: ClusterConfig) -> ExpertPlacement:
    """Contiguous EP placement: expert e lives on rank e // experts_per_rank."""
    epr = config.experts_per_rank
    return ExpertPlacement(tuple((e // epr,) for e in range(config.total_experts)), 0)


def _even_shares(count: int, parts: int) -> list[int]:
    q, r = divmod(count, parts)
    return [q + (i < r) for i in range(parts)]


def aggregate_rank_loads(
    expert_loads: Mapping[int, tuple[int, int]],
    placement: ExpertPlacement,
    num_ranks: int,
) -> list[RankLoad]:
    """Per-rank (vision, text) sums of per-expert counts; replicas split evenly with
    the remainder on the lowest rank ids (core.py:106-130)."""
    acc = np.zeros((num_ranks, 2), dtype=np.int64)
    for expert, (v, t) in expert_loads.items():
        if not 0 <= expert < placement.num_experts:
            raise PlacementMismatchError(f"expert {expert} not in placement")
        hosts = sorted(set(placement.assignment[expert]))
        if len(hosts) == 1:
            acc[hosts[0]] += (v, t)
            continue
        for h, sv, st in zip(hosts, _even_shares(v, len(hosts)), _even_shares(t, len(hosts))):
            acc[h] += (sv, st)
    return [RankLoad(r, int(acc[r, 0]), int(acc[r, 1])) for r in range(num_ranks)]


def rank_loads_from_counts(expert_vt: np.ndarray, config: ClusterConfig) -> list[RankLoad]:
    """Fast path for the static placement: ``expert_vt`` is the [E, 2] (vision, text)
    pair-count array produced by the router kernel (realb_moe_align)."""
    vt = np.asarray(expert_vt, dtype=np.int64).reshape(config.num_ranks, config.experts_per_rank, 2)
    s = vt.sum(axis=1)
    return [RankLoad(r, int(s[r, 0]), int(s[r, 1])) for r in range(config.num_ranks)]


@dataclass(frozen=True)
class PrecisionPlan:
    per_rank_precision: tuple[Precision, ...]
    hot_ranks: frozenset[int]
    vision_heavy_ranks: frozenset[int]
    active: bool

    def __post_init__(self):
        if not self.active and any(p is Precision.W4A4 for p in self.per_rank_precision):
            raise ValueError("inactive plan must be all W16A16")

    def expert_precision(self, placement: ExpertPlacement) -> np.ndarray:
        """uint8 [E] precision code per expert (expanded through the placement)."""
        out = np.zeros(placement.num_experts, dtype=np.uint8)
        for e, hosts in enumerate(placement.assignment):
            out[e] = self.per_rank_precision[hosts[0]].code
        return out

    @property
    def accelerated_ranks(self) -> frozenset[int]:
        return frozenset(r for r, p in enumerate(self.per_rank_precision) if p is Precision.W4A4)


@dataclass(frozen=True)
class RealbParams:
    capacity_factor: float = 1.0       # C
    modality_threshold: float = 0.7    # M_d
    global_batch_threshold: int = 2048

    def __post_init__(self):
        if self.capacity_factor <= 0:
            raise ValueError("capacity_factor must be > 0")
        if not 0.0 <= self.modality_threshold <= 1.0:
            raise ValueError("modality_threshold must lie in [0, 1]")
        if self.global_batch_threshold < 0:
            raise ValueError("global_batch_threshold must be >= 0")


def plan_baseline(loads: Sequence[RankLoad]) -> PrecisionPlan:
    if not loads:
        raise ValueError("loads must be non-empty")
    return PrecisionPlan((Precision.W16A16,) * len(loads), frozenset(), frozenset(), False)


def plan_fp4_all(loads: Sequence[RankLoad]) -> PrecisionPlan:
    if not loads:
        raise ValueError("loads must be non-empty")
    every = frozenset(range(len(loads)))
    return PrecisionPlan((Precision.W4A4,) * len(loads), every, every, True)


def plan_realb(loads: Sequence[RankLoad], params: RealbParams, config: ClusterConfig) -> PrecisionPlan:
    """W4A4 on ranks that are hot (load > C x mean) and vision-heavy (v/total > M_d;
    any loaded rank when modality-isolated), gated on the global batch size."""
    if len(loads) != config.num_ranks:
        raise ValueError("loads length must equal num_ranks")
    R = len(loads)
    vt = np.array([[l.vision_tokens, l.text_tokens] for l in loads], dtype=np.int64)
    prec = np.zeros(R, dtype=np.uint8)
    flags = np.zeros(R, dtype=np.uint8)
    active = _lib.call(
        "realb_plan", vt.ctypes.data_as(C.c_void_p), R, float(params.capacity_factor),
        float(params.modality_threshold), int(params.global_batch_threshold),
        int(bool(config.modality_isolated)), prec.ctypes.data_as(C.c_void_p),
        flags.ctypes.data_as(C.c_void_p))
    if not active:
        return plan_baseline(loads)
    # the C routine flags list positions; the reference collects the hot and
    # vision-heavy sets by RankLoad.rank and indexes precision by rank id
    # (balancers.py:104-118), so the sets are mapped back through l.rank
    hot = frozenset(int(loads[i].rank) for i in np.flatnonzero(flags & 1))
    vision = frozenset(int(loads[i].rank) for i in np.flatnonzero(flags & 2))
    accelerated = hot & vision
    return PrecisionPlan(
        tuple(Precision.W4A4 if r in accelerated else Precision.W16A16 for r in range(R)),
        hot,
        vision,
        True,
    )


def plan_for(strategy: str, loads: Sequence[RankLoad], config: ClusterConfig,
             realb_params: RealbParams | None = None) -> PrecisionPlan:
    """Per-layer plan for a strategy tag; EPLB variants never touch precision."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; valid: {', '.join(STRATEGIES)}")
    if strategy == "fp4all":
        return plan_fp4_all(loads)
    if strategy in ("realb", "realb-seq"):
        return plan_realb(loads, realb_params or RealbParams(), config)
    return plan_baseline(loads)
