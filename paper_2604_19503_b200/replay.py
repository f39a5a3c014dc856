"""Trace-driven routing replay and the measured-timing bridge.

The reference drives its "MoE layer" from per-(iteration, layer, expert)
(vision, text) token-count traces (``moesim/tracegen.py``: ``IterationTrace``
:69-103, ``read_trace``/``write_trace`` :255-278) and writes per-run results
as ``layers.csv`` / ``ranks.csv`` / ``events.csv`` / ``summary.json``
(``engine.py:258-288``, ``cli.py:90-123``) that ``moesim compare``
(``cli.py:157-185``, ``metrics.speedup_report`` :143-165) turns into speedups.

This module executes such a trace on the GPU:

* ``routing_from_expert_loads`` turns one layer's per-expert counts into a
  token batch — a modality mask and k distinct experts per token — whose
  per-expert (token, expert) pair counts are exactly ``k x`` the trace's
  (each trace token is routed to k experts; D2 in DESIGN.md). The hidden states
  are built with routing margins (``workload.make_hidden``) so the real
  router kernel selects exactly those experts, and the device-side counts,
  per-rank loads and plan can be checked against the reference's
  ``aggregate_rank_loads`` + ``plan_for`` on the same records.
* ``MeasuredRun`` has ``RunResult``'s shape (engine.py:89-115) with
  ``LayerTiming``s filled from CUDA-event measurements, and ``write_run``
  writes the reference's file schemas so the unmodified ``moesim compare`` can
  read hardware runs.
"""

from __future__ import annotations

import csv
import hashlib
import json
import os
from dataclasses import dataclass, field
from typing import Mapping

import numpy as np

from .moe import LayerTiming, PipelineMode
from .policy import (ClusterConfig, Precision, PrecisionPlan, RankLoad, RealbParams,
                     STRATEGIES, aggregate_rank_loads, place_experts_static, plan_for)

TRACE_HEADER = "iter,layer,expert,vision_tokens,text_tokens"  # tracegen.py:30


class TraceParseError(ValueError):
    """Malformed trace file (tracegen.py, read_trace)."""


class TraceMismatchError(ValueError):
    """Trace records inconsistent with the cluster (tracegen.py, IterationTrace)."""


@dataclass(frozen=True)
class IterationTrace:
    """Per (iteration, layer, expert) (vision, text) counts (tracegen.py:69-103)."""

    records: tuple[tuple[int, int, int, int, int], ...]
    cluster: ClusterConfig

    def __post_init__(self):
        seen = set()
        for it, layer, expert, v, t in self.records:
            if not 0 <= layer < self.cluster.num_layers:
                raise TraceMismatchError(f"layer {layer} out of range")
            if not 0 <= expert < self.cluster.total_experts:
                raise TraceMismatchError(f"expert {expert} out of range")
            if it < 0 or v < 0 or t < 0:
                raise TraceMismatchError("negative field in trace record")
            if (it, layer, expert) in seen:
                raise TraceMismatchError(f"duplicate record for {(it, layer, expert)}")
            seen.add((it, layer, expert))
        index: dict = {}
        for it, la, e, v, t in self.records:
            index.setdefault((it, la), {})[e] = (v, t)
        object.__setattr__(self, "_index", index)

    @property
    def num_iterations(self) -> int:
        return 1 + max((r[0] for r in self.records), default=-1)

    def layer_loads(self, iteration: int, layer: int) -> dict[int, tuple[int, int]]:
        return self._index.get((iteration, layer), {})


def read_trace(path, config: ClusterConfig) -> IterationTrace:
    """tracegen.py:262-278 file format and errors."""
    with open(path, "r", encoding="utf-8") as f:
        lines = f.read().splitlines()
    if not lines or lines[0] != TRACE_HEADER:
        raise TraceParseError(f"{path}: line 1: bad or missing header")
    records = []
    for lineno, line in enumerate(lines[1:], start=2):
        parts = line.split(",")
        if len(parts) != 5:
            raise TraceParseError(f"{path}: line {lineno}: expected 5 fields")
        try:
            records.append(tuple(int(p) for p in parts))
        except ValueError:
            raise TraceParseError(f"{path}: line {lineno}: non-integer field") from None
    return IterationTrace(tuple(records), config)


def write_trace(trace: IterationTrace, path) -> None:
    lines = [TRACE_HEADER] + [",".join(str(x) for x in rec) for rec in sorted(trace.records)]
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def file_sha256(path) -> str:
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


# ----------------------------------------------------------------------------- routing
def _waterfill(target: np.ndarray, cap: int, group: np.ndarray) -> np.ndarray:
    """Integer counts <= cap with the same per-group sums as ``target``: the
    excess of experts above the cap is spread over the other experts of the
    same group (EP rank), most headroom first."""
    out = np.minimum(target, cap).astype(np.int64)
    for g in np.unique(group):
        m = np.flatnonzero(group == g)
        excess = int(target[m].sum() - out[m].sum())
        while excess > 0:
            room = cap - out[m]
            open_ = m[room > 0]
            if len(open_) == 0:
                raise ValueError(f"rank {int(g)} load exceeds what top-k routing can place on its experts")
            share = -(-excess // len(open_))
            for e in open_[np.argsort(-(cap - out[open_]), kind="stable")]:
                add = min(share, cap - int(out[e]), excess)
                out[e] += add
                excess -= add
                if excess == 0:
                    break
    return out


def routing_from_expert_loads(loads: Mapping[int, tuple[int, int]], num_experts: int, k: int,
                              experts_per_rank: int | None = None,
                              seed: int = 2024) -> tuple[np.ndarray, np.ndarray]:
    """(modality uint8 [T], idx int32 [T, k]) with T = sum(v + t) tokens, every
    token routed to k distinct experts, and per-rank (vision, text) pair loads
    exactly k x the trace's (each trace token becomes one top-k token; D2).

    Per expert the pair count is k x the trace count, except that top-k routing
    can place at most one pair per token on an expert: an expert above that
    (the reference's top-1-semantics traces give the hottest expert up to ~20 %
    of a modality) is capped and its excess spread over the other experts of
    its EP rank (``_waterfill``), so rank loads — what the policy sees — stay
    exact. With ``experts_per_rank=None`` no capping is allowed (ValueError).

    Per modality the list of expert ids, expert e repeated c_e times in id
    order, is dealt column-wise: token j takes entries j, j+n, ..., j+(k-1)n
    (n = tokens of that modality); a contiguous run of length c_e <= n never
    hits one token twice. Tokens are then shuffled (seeded)."""
    counts = np.zeros((num_experts, 2), np.int64)
    for e, (v, t) in loads.items():
        if not 0 <= e < num_experts:
            raise TraceMismatchError(f"expert {e} out of range")
        counts[e] = (v, t)
    mods, idxs = [], []
    for m, col in ((1, 0), (0, 1)):
        n = int(counts[:, col].sum())
        if n == 0:
            continue
        c = k * counts[:, col]
        if int(c.max()) > n:
            if experts_per_rank is None:
                raise ValueError(f"expert {int(c.argmax())} needs {int(c.max())} of {n} "
                                 f"{'vision' if m else 'text'} tokens: not routable top-{k}")
            c = _waterfill(c, n, np.arange(num_experts) // experts_per_rank)
        lst = np.repeat(np.arange(num_experts, dtype=np.int32), c)
        idxs.append(lst.reshape(k, n).T)
        mods.append(np.full(n, m, np.uint8))
    if not idxs:
        return np.zeros(0, np.uint8), np.zeros((0, k), np.int32)
    idx = np.concatenate(idxs)
    mod = np.concatenate(mods)
    perm = np.random.default_rng(seed).permutation(len(mod))
    return mod[perm], np.ascontiguousarray(idx[perm])


def replay_pair_counts(mod: np.ndarray, idx: np.ndarray, num_experts: int) -> np.ndarray:
    """[E, 2] (vision, text) pair counts of a replayed batch."""
    vis = np.repeat(mod, idx.shape[1]) == 1
    e = idx.reshape(-1).astype(np.int64)
    return np.stack([np.bincount(e[vis], minlength=num_experts),
                     np.bincount(e[~vis], minlength=num_experts)], axis=1)


def pair_loads(loads: Mapping[int, tuple[int, int]], k: int) -> dict[int, tuple[int, int]]:
    """The (token, expert)-pair counts a replayed layer produces (k x the trace)."""
    return {e: (k * v, k * t) for e, (v, t) in loads.items()}


# ----------------------------------------------------------------------------- measured run
@dataclass(frozen=True)
class MigrationEvent:
    """engine.py:89-94: one EPLB rebalance's replica moves and the stall charged."""

    iteration: int
    replicas_moved: int
    volume_bytes: int
    charged_ns: int


@dataclass
class MeasuredRun:
    """``RunResult`` (engine.py:89-115) filled from measurements."""

    strategy: str
    layer_timings: dict = field(default_factory=dict)
    plans: dict = field(default_factory=dict)
    migration_events: list = field(default_factory=list)
    max_redundant_count: int = 0
    timing_source: str = ""

    @property
    def e2e_time_ns(self) -> int:
        return sum(t.layer_latency_ns for t in self.layer_timings.values()) + \
            sum(e.charged_ns for e in self.migration_events)

    @property
    def compute_only_total_ns(self) -> int:
        return sum(t.compute_only_ns for t in self.layer_timings.values())

    @property
    def migration_volume_bytes(self) -> int:
        return sum(e.volume_bytes for e in self.migration_events)


def text_exposure(run: MeasuredRun, trace: IterationTrace) -> float:
    """metrics.py:72-90: text tokens on W4A4 ranks / all text tokens."""
    cfg = trace.cluster
    placement = place_experts_static(cfg)
    exposed = total = 0
    for (it, layer), plan in run.plans.items():
        for rank, load in enumerate(aggregate_rank_loads(trace.layer_loads(it, layer), placement, cfg.num_ranks)):
            total += load.text_tokens
            if plan.per_rank_precision[rank] is Precision.W4A4:
                exposed += load.text_tokens
    return exposed / total if total else 0.0


def _mem_delta(run: MeasuredRun, config: ClusterConfig) -> int:
    """metrics.summarize_run's memory delta (metrics.py:105-129 via
    costmodel.memory_overhead): it depends only on the replica count."""
    lb = config.num_layers * config.bytes_per_expert  # costmodel.py:105-111 operation order
    E = config.total_experts
    return round(lb * (E + run.max_redundant_count) / config.num_ranks) - round(lb * E / config.num_ranks)


def write_run(run: MeasuredRun, trace: IterationTrace, out_dir, trace_sha256: str,
              ranks_iters=(0,)) -> dict:
    """layers.csv / ranks.csv / events.csv / summary.json in the reference's
    schemas (engine.py:258-288, cli.py:102-123)."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "layers.csv"), "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["iter", "layer", "strategy", "mode", "latency_ns", "compute_only_ns", "critical_rank"])
        for (it, layer), t in sorted(run.layer_timings.items()):
            w.writerow([it, layer, run.strategy, t.pipeline_mode.value, t.layer_latency_ns, t.compute_only_ns,
                        t.critical_rank])
    with open(os.path.join(out_dir, "ranks.csv"), "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["iter", "layer", "rank", "schedule_ns", "transform_ns", "dispatch_ns", "compute_ns",
                    "combine_ns", "total_ns"])
        for (it, layer), t in sorted(run.layer_timings.items()):
            if it not in ranks_iters:
                continue
            for rank, p in enumerate(t.per_rank):
                w.writerow([it, layer, rank, p.schedule_ns, p.transform_ns, p.dispatch_ns, p.compute_ns,
                            p.combine_ns, t.per_rank_total_ns[rank]])
    with open(os.path.join(out_dir, "events.csv"), "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["iter", "replicas_moved", "volume_bytes", "charged_ns"])
        for e in run.migration_events:
            w.writerow([e.iteration, e.replicas_moved, e.volume_bytes, e.charged_ns])
    meta = {
        "strategy": run.strategy,
        "trace_sha256": trace_sha256,
        "e2e_time_ns": run.e2e_time_ns,
        "compute_only_total_ns": run.compute_only_total_ns,
        "mem_delta_bytes": _mem_delta(run, trace.cluster),
        "migration_bytes": run.migration_volume_bytes,
        "text_exposure": text_exposure(run, trace),
        "timing_source": run.timing_source,
    }
    with open(os.path.join(out_dir, "summary.json"), "w") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return meta


def speedup_report(summaries: Mapping[str, Mapping]) -> list[dict]:
    """metrics.py:143-165 over summary.json dicts (layer = compute-only, e2e = full path)."""
    if "baseline" not in summaries:
        raise ValueError("speedup report requires a baseline run")
    base = summaries["baseline"]
    return [{"strategy": n,
             "layer_speedup": base["compute_only_total_ns"] / s["compute_only_total_ns"],
             "e2e_speedup": base["e2e_time_ns"] / s["e2e_time_ns"],
             "mem_delta_bytes": s["mem_delta_bytes"], "migration_bytes": s["migration_bytes"],
             "text_exposure": s["text_exposure"]} for n, s in sorted(summaries.items())]


# ----------------------------------------------------------------------------- GPU replay
class TraceReplay:
    """Replays a trace layer by layer on cuda:0 as virtual EP-R (R = the trace's
    cluster): per layer, the real router/plan/dispatch/GEMM/combine forward runs
    on the replayed batch, the device plan is cross-checked against the host
    policy on the trace's own loads, and each strategy's per-rank phases are
    measured (virtual_ep.measure_phases) into a ``LayerTiming``."""

    def __init__(self, torch, config: str, trace: IterationTrace, params: RealbParams | None = None,
                 seed: int = 2024):
        from . import _lib
        from .moe import SHAPES, MoELayer, MoEWeights
        from .workload import WorkloadSpec, make_experts, make_router

        self.torch, self.trace = torch, trace
        self.shape = shape = SHAPES[config]
        cl = trace.cluster
        if cl.total_experts != shape.num_experts:
            raise TraceMismatchError(f"trace has {cl.total_experts} experts, {shape.name} has {shape.num_experts}")
        self.cluster = ClusterConfig(cl.num_ranks, 1, cl.experts_per_rank, cl.bytes_per_expert,
                                     shape.modality_isolated or cl.modality_isolated)
        k = shape.top_k
        self.params = params or RealbParams()
        # D2: the device counts (token, expert) pairs = k x the trace's tokens; the gate scales with k
        self.pair_params = RealbParams(self.params.capacity_factor, self.params.modality_threshold,
                                       self.params.global_batch_threshold * k)
        self.seed = seed
        max_t = max(sum(v + t for v, t in trace.layer_loads(it, la).values())
                    for it in range(trace.num_iterations) for la in range(cl.num_layers))
        self.unit, router = make_router(shape, WorkloadSpec(tokens=1, seed=seed))
        gu, dn = make_experts(shape)
        bias = torch.zeros(shape.num_experts, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
        self.layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn, bias=bias), max_tokens=max_t,
                              cluster=self.cluster)
        del gu, dn

    def batch(self, it: int, la: int):
        from .workload import WorkloadSpec, make_hidden

        loads = self.trace.layer_loads(it, la)
        mod, idx = routing_from_expert_loads(loads, self.shape.num_experts, self.shape.top_k,
                                             self.cluster.experts_per_rank, seed=self.seed + 7919 * it + la)
        spec = WorkloadSpec(tokens=len(mod), seed=self.seed, layer=la, rank=it)
        x = make_hidden(self.shape, spec, self.unit, idx)
        return x, self.torch.from_numpy(mod).cuda(), idx

    def run(self, strategies=("baseline", "fp4all", "realb"), iterations=None, check=True,
            eplb_state: dict | None = None):
        """-> ({strategy: MeasuredRun}, [per-layer parity checks]).

        "eplb" / "async-eplb" run the reference's replication balancer
        (eplb.py, balancers.py:143-199) on the replayed loads: at an iteration
        whose rebalance is due (engine.py:181-205) the placement is rebuilt and
        the moved replicas' weight bytes are charged as a migration over NVLink
        (all of it for eplb, the part exceeding that iteration's dispatch time for
        async-eplb, engine.py:217-228); each rank's BF16 compute over its hosted
        replica shares (rank_expert_rows) is measured on the GPU. ``eplb_state``:
        EplbState keyword arguments (default: the reference's, window 100 /
        interval 100 / budget 8)."""
        from .eplb import EplbState, eplb_schedule, rank_expert_rows
        from .virtual_ep import (NVLINK_GBPS, a2a_ms, layer_timing, measure_arms, measure_rank_compute,
                                 measure_transform, placement_compute_arm, traffic_matrix)

        torch, cl, shape = self.torch, self.cluster, self.shape
        for s in strategies:
            if s not in STRATEGIES:
                raise ValueError(f"unknown strategy {s!r}; valid: {', '.join(STRATEGIES)}")
        src = ("measured per-rank compute + K3 (CUDA events, virtual EP on one B200) + NVLink model for "
               "dispatch/combine/migration")
        runs = {s: MeasuredRun(s, timing_source=src) for s in strategies}
        checks = []
        R, epr, E, H, k = cl.num_ranks, cl.experts_per_rank, shape.num_experts, shape.hidden, shape.top_k
        static = place_experts_static(cl)
        its = range(self.trace.num_iterations) if iterations is None else iterations
        precision_strats = [s for s in strategies if s not in ("eplb", "async-eplb")]
        eplb_strats = [s for s in strategies if s in ("eplb", "async-eplb")]
        # forward order: all-BF16 rows first, then the NVFP4 strategies, so every
        # strategy's per-rank compute reads operands a forward actually produced
        order = sorted(set(precision_strats) | ({"baseline"} if eplb_strats else set()),
                       key=lambda s: {"fp4all": 1, "realb": 2, "realb-seq": 2}.get(s, 0))
        # placements per iteration (a pure function of the trace's totals)
        sched = {s: dict(zip(its, eplb_schedule(self.trace, EplbState(**(eplb_state or {})), its)))
                 for s in eplb_strats}
        eplace = {}
        # a migrated replica moves the expert's real weights: gate, up, down in bf16
        bytes_per_expert = 3 * H * shape.intermediate * 2
        for it in its:
            pending = {}
            for s in eplb_strats:  # engine.py:181-205
                eplace[s], moved = sched[s][it]
                runs[s].max_redundant_count = max(runs[s].max_redundant_count, eplace[s].redundant_count)
                if moved is not None:
                    vol = moved * bytes_per_expert
                    pending[s] = (moved, vol, int(round(vol / (NVLINK_GBPS * 1e9) * 1e9)))
            dispatch_total = {s: 0 for s in eplb_strats}
            for la in range(self.trace.cluster.num_layers):
                loads = self.trace.layer_loads(it, la)
                if not loads:
                    raise TraceMismatchError(f"iteration {it} has no records for layer {la}")
                x, mod, idx = self.batch(it, la)
                T = x.shape[0]
                want = replay_pair_counts(mod.cpu().numpy(), idx, E)
                plans, precs = {}, {}
                for s in order:
                    res = self.layer.forward(x, mod, s, self.pair_params)
                    torch.cuda.synchronize()
                    plans[s] = plan = res.plan
                    precs[s] = plan.expert_precision(static).astype(np.int64)
                    if check:
                        host_pairs = plan_for(s, aggregate_rank_loads(pair_loads(loads, k), static, R), cl,
                                              self.pair_params)
                        host_trace = plan_for(s, aggregate_rank_loads(loads, static, R), cl, self.params)
                        checks.append({"iter": it, "layer": la, "strategy": s, "tokens": T,
                                       "counts_equal": bool((res.expert_vt.astype(np.int64) == want).all()),
                                       "routing_equal": bool((np.sort(self.layer.topk_idx[:T].cpu().numpy(), 1)
                                                              == np.sort(idx, 1)).all()),
                                       "plan_equal_pairs": plan == host_pairs,
                                       "plan_equal_trace": plan == host_trace,
                                       "plan": [p.value for p in plan.per_rank_precision],
                                       "host_plan": [p.value for p in host_trace.per_rank_precision],
                                       "w4a4_ranks": sorted(plan.accelerated_ranks)})
                # per-rank compute of every arm, interleaved per rank
                comp = dict(zip(order, measure_rank_compute(torch, self.layer, T, [precs[s] for s in order],
                                                            R, epr, reps=5)))
                T_local = max(1, -(-T // R))
                pairs = traffic_matrix(idx, T_local, epr, R)
                if eplb_strats:
                    expert_pairs = want.sum(1)
                    rows = {s: rank_expert_rows(expert_pairs, eplace[s], R) for s in eplb_strats}
                    ecomp = measure_arms(torch, [placement_compute_arm(torch, self.layer, rows[s])
                                                 for s in eplb_strats], reps=5)
                    comp.update(zip(eplb_strats, ecomp))
                any_fp4 = np.max([precs[s] for s in order], axis=0)
                trans = measure_transform(torch, self.layer, any_fp4, R, epr)
                disp = a2a_ms(pairs, np.full(R, 2.0 * H))
                comb = a2a_ms(pairs.T.copy(), np.full(R, 2.0 * H))
                for s in precision_strats:
                    acc = [bool(precs[s][r * epr] == 1) for r in range(R)]
                    mode = PipelineMode.OVERLAPPED if s in ("fp4all", "realb") and plans[s].active \
                        else PipelineMode.SEQUENTIAL  # engine.py:162-167
                    tr = [trans[r] if acc[r] else 0.0 for r in range(R)]
                    runs[s].plans[(it, la)] = plans[s]
                    runs[s].layer_timings[(it, la)] = layer_timing(comp[s], tr, acc, mode, disp, comb)
                for s in eplb_strats:
                    # source rank x expert pairs, sent to the expert's hosts in their shares
                    src_e = np.zeros((R, E), np.float64)
                    np.add.at(src_e, (np.repeat(np.arange(T) // T_local, k), idx.reshape(-1)), 1.0)
                    share = rows[s] / np.maximum(expert_pairs, 1)[None, :]      # [R_dst, E]
                    traffic = src_e @ share.T                                      # [R_src, R_dst]
                    d_s = a2a_ms(traffic, np.full(R, 2.0 * H))
                    c_s = a2a_ms(traffic.T.copy(), np.full(R, 2.0 * H))
                    lt = layer_timing(comp[s], [0.0] * R, [False] * R, PipelineMode.SEQUENTIAL, d_s, c_s)
                    runs[s].plans[(it, la)] = plan_for(s, aggregate_rank_loads(loads, static, R), cl, self.params)
                    runs[s].layer_timings[(it, la)] = lt
                    dispatch_total[s] += lt.per_rank[0].dispatch_ns
            for s in eplb_strats:  # migration charge (engine.py:217-228), then observe
                if s in pending:
                    moved, vol, mig_ns = pending[s]
                    charged = max(0, mig_ns - dispatch_total[s]) if s == "async-eplb" else mig_ns
                    runs[s].migration_events.append(MigrationEvent(it, moved, vol, charged))
        return {s: runs[s] for s in strategies}, checks
