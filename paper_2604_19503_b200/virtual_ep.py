"""Virtual expert parallelism on one GPU: the ReaLB policy effect, measured.

With one GPU the real plan is never active (R = 1, balancers.py:103-104). This
module runs the EP-R layer's *global* batch (R x tokens-per-GPU) on one device
with the plan evaluated over R virtual ranks, then times every virtual rank's
expert computation in isolation (its own grouped-GEMM launches over only its
experts' rows). The layer's compute-only latency is the max over ranks, the
definition of ``LayerTiming.compute_only_ns`` (engine.py:156) and of the
paper's layer latency with dispatch/combine excluded.

Communication is not executed on one GPU; the full-path figure fills the
reference ``RankPhases`` schema with the measured compute / transform times
and a stated NVLink projection for dispatch/combine (bytes each rank receives
/ 770 GB/s measured peer bandwidth + 10 us), i.e. engine.py's overlap rule with
measured terms where measurement exists. It is labelled a projection.
"""

from __future__ import annotations

import numpy as np

from .moe import SHAPES, LayerTiming, MoELayer, MoEWeights, PipelineMode, RankPhases
from .policy import ClusterConfig, RealbParams

NVLINK_GBPS = 770.0   # measured per-direction peer copy (B200_PROFILING.md)
ALPHA_US = 10.0


def _median_ms(torch, fn, reps=7):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return float(sorted(ts)[len(ts) // 2])


def virtual_ep_report(args, torch, R: int = 8) -> dict:
    from . import _lib
    from .workload import WorkloadSpec, make_batch, make_experts

    shape = SHAPES[args.config]
    E, H = shape.num_experts, shape.hidden
    if E % R:
        return {"skipped": f"{E} experts not divisible by {R}"}
    T = args.tokens * R
    spec = WorkloadSpec(tokens=T, vision_frac=args.vision_frac, num_ranks=R)
    x, mod, router, _ = make_batch(shape, spec)
    gu, dn = make_experts(shape)
    bias = torch.zeros(E, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
    w = MoEWeights.from_hf(shape, router, gu, dn, bias=bias)
    del gu, dn
    epr = E // R
    cluster = ClusterConfig(R, 1, epr, 1, shape.modality_isolated)
    layer = MoELayer(w, max_tokens=T, cluster=cluster)
    params = RealbParams()

    res = layer.forward(x, mod, "realb", params)
    torch.cuda.synchronize()
    plan = res.plan
    prec = plan.expert_precision(layer.placement).astype(np.int64)
    vt = res.expert_vt.astype(np.int64)
    rank_vt = vt.reshape(R, epr, 2).sum(1)

    def per_rank(p_full):
        out = []
        for r in range(R):
            m = np.full(E, 2, np.int64)
            m[r * epr:(r + 1) * epr] = p_full[r * epr:(r + 1) * epr]
            out.append(_median_ms(torch, lambda: layer.expert_compute(T, m)))
        return out

    realb_ms = per_rank(prec)
    transform_ms = [0.0] * R
    for r in range(R):
        if prec[r * epr] == 1:
            transform_ms[r] = _median_ms(torch, lambda: layer.quantize_experts(range(r * epr, (r + 1) * epr)))
    whole_realb = _median_ms(torch, lambda: layer.forward(x, mod, "realb", params), reps=5)
    layer.forward(x, mod, "baseline")
    torch.cuda.synchronize()
    bf16_ms = per_rank(np.zeros(E, np.int64))
    whole_bf16 = _median_ms(torch, lambda: layer.forward(x, mod, "baseline"), reps=5)

    # projected full path: engine.py:120-159 overlap rule with measured compute/transform
    recv_bytes = rank_vt.sum(1) * (R - 1) / R * H * 2  # pairs from remote ranks, bf16 rows
    disp_ms = [ALPHA_US / 1e3 + b / (NVLINK_GBPS * 1e9) * 1e3 for b in recv_bytes]
    sched_ms = ALPHA_US / 1e3

    def timing(comp, trans, accelerated, mode):
        phases, totals = [], []
        worst = max(disp_ms)  # globally synchronised all-to-all: every rank waits for the slowest
        for r in range(R):
            ph = RankPhases(int(sched_ms * 1e6), int(trans[r] * 1e6), int(worst * 1e6), int(comp[r] * 1e6),
                            int(worst * 1e6))
            phases.append(ph)
            totals.append(ph.total(mode, accelerated[r]))
        lat = max(totals)
        return LayerTiming(tuple(phases), tuple(totals), lat, max(p.compute_ns for p in phases),
                           totals.index(lat), mode)

    acc = [bool(prec[r * epr] == 1) for r in range(R)]
    lt_realb = timing(realb_ms, transform_ms, acc, PipelineMode.OVERLAPPED if plan.active else PipelineMode.SEQUENTIAL)
    lt_bf16 = timing(bf16_ms, [0.0] * R, [False] * R, PipelineMode.SEQUENTIAL)
    return {
        "what": f"EP{R} emulated on 1 GPU: global batch {T} tokens, plan over {R} virtual ranks, "
                "per-rank expert compute timed in isolation (layer = max over ranks)",
        "plan_w4a4_ranks": sorted(plan.accelerated_ranks), "hot_ranks": sorted(plan.hot_ranks),
        "vision_heavy_ranks": sorted(plan.vision_heavy_ranks),
        "rank_pairs": rank_vt.sum(1).tolist(),
        "rank_vision_ratio": [round(float(a / max(1, a + b)), 3) for a, b in rank_vt],
        "per_rank_compute_ms": {"bf16": bf16_ms, "realb": realb_ms},
        "transform_ms": transform_ms,
        "compute_only_ms": {"bf16": max(bf16_ms), "realb": max(realb_ms)},
        "compute_only_speedup": max(bf16_ms) / max(realb_ms),
        "one_gpu_whole_layer_ms": {"bf16": whole_bf16, "realb": whole_realb},
        "projected_full_path_ms": {"bf16": lt_bf16.layer_latency_ns / 1e6, "realb": lt_realb.layer_latency_ns / 1e6,
                                   "model": f"dispatch=combine={ALPHA_US}us + max_r recv_bytes_r/{NVLINK_GBPS}GB/s"},
        "projected_full_path_speedup": lt_bf16.layer_latency_ns / lt_realb.layer_latency_ns,
        "transform_hidden": all(t <= max(disp_ms) for t in transform_ms),
    }
