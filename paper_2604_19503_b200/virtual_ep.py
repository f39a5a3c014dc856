"""Virtual expert parallelism on one GPU: the ReaLB policy effect, measured.

With one GPU the real plan is never active (R = 1, balancers.py:103-104). This
module runs the EP-R layer's *global* batch (R x tokens-per-GPU) on one device
with the plan evaluated over R virtual ranks, then times every virtual rank's
expert computation in isolation (its own grouped-GEMM launches over only its
experts' rows). The layer's compute-only latency is the max over ranks, the
definition of ``LayerTiming.compute_only_ns`` (engine.py:156) and of the
paper's layer latency with dispatch/combine excluded.

Communication is not executed on one GPU. The full-path figure fills the
reference ``RankPhases`` schema with the measured compute / transform times and
a stated NVLink projection for dispatch and combine: the exact per-rank send and
receive bytes of this batch's routing (token t lives on rank t // T_local,
pair (t, e) goes to rank e // experts_per_rank) over 770 GB/s measured peer
bandwidth + 10 us, every all-to-all finishing with its slowest rank; then
engine.py's overlap rule (RankPhases.total, engine.py:63-76). It is labelled a
projection. With ``fp4_dispatch`` the rows bound for W4A4 ranks travel as NVFP4
(H/2 code bytes + H/16 scale bytes instead of 2H).
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


def traffic_matrix(idx: np.ndarray, T_local: int, epr: int, R: int) -> np.ndarray:
    """pairs[src_rank, dst_rank] of one layer's dispatch (DP tokens, contiguous EP)."""
    src = np.repeat(np.arange(idx.shape[0]) // T_local, idx.shape[1])
    dst = idx.reshape(-1).astype(np.int64) // epr
    return np.bincount(src * R + dst, minlength=R * R).reshape(R, R)


def a2a_ms(pairs: np.ndarray, row_bytes_to: np.ndarray) -> float:
    """One all-to-all over NVLink: every rank's max(send, receive) bytes (self
    traffic excluded) / peer bandwidth, finishing with the slowest rank."""
    R = pairs.shape[0]
    off = pairs * (1 - np.eye(R, dtype=pairs.dtype))
    bytes_ = off * row_bytes_to[None, :]
    per_rank = np.maximum(bytes_.sum(1), bytes_.sum(0))
    return ALPHA_US / 1e3 + float(per_rank.max()) / (NVLINK_GBPS * 1e9) * 1e3


def measure_arms(torch, arms, reps: int = 7):
    """arms[a][r]: a callable launching arm a's work for virtual rank r. Per rank,
    the arms are timed interleaved per repetition (clock / power drift hits every
    arm alike); returns [arm][rank] median ms."""
    R = len(arms[0])
    out = [[0.0] * R for _ in arms]
    for r in range(R):
        ts = [[] for _ in arms]
        for _ in range(reps):
            for a, arm in enumerate(arms):
                ts[a].append(_median_ms(torch, arm[r], reps=1))
        for a in range(len(arms)):
            out[a][r] = float(sorted(ts[a])[len(ts[a]) // 2])
    return out


def measure_rank_compute(torch, layer, T: int, precs, R: int, epr: int, reps: int = 7):
    """Per virtual rank, the expert compute of that rank's experts alone (their
    grouped-GEMM launches over the rows the last forward dispatched), for each
    expert-precision vector in ``precs`` (codes 0 W16A16 / 1 W4A4)."""
    E = R * epr
    arms = []
    for p in precs:
        arm = []
        for r in range(R):
            m = np.full(E, 2, np.int64)
            m[r * epr:(r + 1) * epr] = p[r * epr:(r + 1) * epr]
            arm.append(lambda m=m: layer.expert_compute(T, m))
        arms.append(arm)
    return measure_arms(torch, arms, reps)


def placement_compute_arm(torch, layer, rank_rows: np.ndarray):
    """Callables timing each rank's BF16 expert compute over its hosted expert
    instances (rank_rows [R, E] pairs, e.g. eplb.rank_expert_rows)."""
    from .moe import host_layout

    arm = []
    for r in range(rank_rows.shape[0]):
        lay, _ = host_layout(rank_rows[r], np.zeros(rank_rows.shape[1], np.int64))
        lt = torch.from_numpy(lay).to(layer.device)
        arm.append(lambda lt=lt: layer.bf16_compute_on(lt))
    return arm


def measure_transform(torch, layer, prec, R: int, epr: int) -> list[float]:
    """K3 time per rank: quantising that rank's experts (0 on W16A16 ranks)."""
    out = [0.0] * R
    for r in range(R):
        if prec[r * epr] == 1:
            out[r] = _median_ms(torch, lambda: layer.quantize_experts(range(r * epr, (r + 1) * epr)))
    return out


def layer_timing(comp_ms, trans_ms, accelerated, mode: PipelineMode, disp_ms: float, comb_ms: float,
                 sched_ms: float = ALPHA_US / 1e3) -> LayerTiming:
    """LayerTiming (engine.py:79-86, :141-159) from per-rank measured compute and
    transform and a globally synchronised dispatch/combine time."""
    phases, totals = [], []
    for r in range(len(comp_ms)):
        ph = RankPhases(int(sched_ms * 1e6), int(trans_ms[r] * 1e6), int(disp_ms * 1e6), int(comp_ms[r] * 1e6),
                        int(comb_ms * 1e6))
        phases.append(ph)
        totals.append(ph.total(mode, accelerated[r]))
    lat = max(totals)
    return LayerTiming(tuple(phases), tuple(totals), lat, max(p.compute_ns for p in phases),
                       totals.index(lat), mode)


class EventMarks:
    """Named CUDA events recorded on given streams (MoELayer.forward(timer=...))."""

    def __init__(self, torch):
        self.torch, self.ev = torch, {}

    def mark(self, name, stream=None):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.ev[name] = e

    def ms(self, a, b):
        return self.ev[a].elapsed_time(self.ev[b])


def measure_k3_overlap(torch, layer, x, mod, params) -> dict:
    """Timeline of one realb forward on this GPU: K3 on the side stream vs the main
    stream's dispatch and BF16 GEMMs, up to the first W4A4 GEMM that needs K3's
    output. stall_ms > 0 would mean the quantiser was NOT hidden."""
    tm = EventMarks(torch)
    layer.forward(x, mod, "realb", params, timer=tm)
    torch.cuda.synchronize()
    if "k3_start" not in tm.ev:
        return {"skipped": "no W4A4 launches for this plan"}
    return {"k3_ms": tm.ms("k3_start", "k3_end"),
            "dispatch_ms": tm.ms("dispatch_start", "dispatch_end"),
            "main_work_before_first_w4a4_gemm_ms": tm.ms("dispatch_start", "fp4_ready"),
            "stall_ms": max(0.0, tm.ms("fp4_ready", "fp4_start")),
            "k3_hidden": tm.ms("k3_end", "fp4_ready") >= 0.0,
            "what": "one-GPU forward of the EP global batch: K3 (side stream) runs under the main "
                    "stream's dispatch and W16A16 GEMMs; stall = wait of the first W4A4 GEMM on K3"}


def measure_ep_kernels(torch, layer, x, mod, T_local: int, recv_rows, w4a4):
    """The EP layer's non-GEMM kernels of every virtual rank, timed on this GPU
    (ep.CudaEPOps runs exactly these around the two all-to-alls):
      send    router + send-side align + pack of the rank's T_local tokens
      recv_r  regroup + row gather of the rows rank r receives (bf16 rows; K4
              quantising gather on a W4A4 rank; packed-NVFP4 gather with fp4 dispatch)
      back_r  index_rows of those rows for the return all-to-all
      combine weighted combine of the rank's T_local tokens
    -> dict of ms (recv* / back lists per rank)."""
    from . import _lib

    dev, H, E, k = layer.device, layer.H, layer.E, layer.k
    n_max = max(1, int(max(recv_rows)))
    u8, i32, bf = torch.uint8, torch.int32, torch.bfloat16
    send = torch.empty(T_local * k * 2 * H, dtype=u8, device=dev)
    pos = torch.empty(T_local, k, dtype=i32, device=dev)
    lay1 = torch.zeros(int(_lib.load().realb_layout_words(E, (T_local + 63) // 64)), dtype=i32, device=dev)
    vt = torch.empty(E, 2, dtype=i32, device=dev)
    zero_prec = torch.zeros(E, dtype=u8, device=dev)
    recv = torch.randn(n_max, H, device=dev).to(bf)
    packed = torch.zeros(n_max, H // 2 + H // 16, dtype=u8, device=dev)
    row_e = torch.zeros(n_max, dtype=i32, device=dev)
    row_p = torch.arange(n_max, dtype=i32, device=dev)
    precs = {0: torch.zeros(E, dtype=u8, device=dev), 1: torch.ones(E, dtype=u8, device=dev)}
    a = torch.empty(n_max, H, dtype=bf, device=dev)
    ac = torch.empty(n_max + 128, H // 2, dtype=u8, device=dev)
    asf = torch.empty((n_max + 128) * H // 16, dtype=u8, device=dev)
    back = torch.empty(n_max, H, dtype=bf, device=dev)
    y = torch.empty(T_local, H, dtype=bf, device=dev)
    fmt = np.zeros(1, np.uint8)
    flag = layer.flag
    xs, ms = x[:T_local], mod[:T_local]

    def sender():
        layer.route(xs, ms)
        sp = _lib.stream_ptr()
        _lib.call("realb_moe_align", layer.chunk_counts.data_ptr(), (T_local + 63) // 64, E,
                  zero_prec.data_ptr(), 1, lay1.data_ptr(), vt.data_ptr(), sp)
        _lib.call("realb_ep_pack", xs.data_ptr(), layer.topk_idx.data_ptr(), T_local, H, E, k,
                  lay1.data_ptr(), (T_local + 63) // 64, 1, fmt.ctypes.data, np.zeros(1, np.int32).ctypes.data,
                  np.zeros(1, np.int64).ctypes.data, pos.data_ptr(), send.data_ptr(), flag.data_ptr(), sp)

    def gather(n, w4, packed_fp4):
        sp = _lib.stream_ptr()
        if packed_fp4:
            return lambda: _lib.call("realb_gather_rows_nvfp4_packed", packed.data_ptr(), row_p.data_ptr(), n,
                                     H, ac.data_ptr(), asf.data_ptr(), None, None, sp)
        return lambda: _lib.call("realb_gather_rows", recv.data_ptr(), row_e.data_ptr(), row_p.data_ptr(), n,
                                 H, 1, precs[int(w4)].data_ptr(), a.data_ptr(), ac.data_ptr(), asf.data_ptr(),
                                 flag.data_ptr(), None, None, sp)

    out = {"send": _median_ms(torch, sender, reps=5)}
    out["recv_bf16"] = [_median_ms(torch, gather(int(n), False, False), reps=5) for n in recv_rows]
    out["recv_w4a4"] = [_median_ms(torch, gather(int(n), True, False), reps=5) if w4a4[r] else 0.0
                        for r, n in enumerate(recv_rows)]
    out["recv_fp4_packed"] = [_median_ms(torch, gather(int(n), True, True), reps=5) if w4a4[r] else 0.0
                              for r, n in enumerate(recv_rows)]
    out["back"] = [_median_ms(torch, lambda n=int(n): _lib.call(
        "realb_index_rows", layer.rows_out.data_ptr(), row_p.data_ptr(), n, H, back.data_ptr(),
        _lib.stream_ptr()), reps=5) for n in recv_rows]
    out["combine"] = _median_ms(torch, lambda: _lib.call(
        "realb_combine", layer.rows_out.data_ptr(), pos.data_ptr(), layer.topk_w.data_ptr(), T_local, H, k,
        None, y.data_ptr(), _lib.stream_ptr()), reps=5)
    return out


def ep_layer_timing(comp_ms, trans_ms, accelerated, mode, disp_a2a, comb_a2a, ek, recv_key_fn):
    """LayerTiming of the EP layer per rank: schedule = router/align/pack + C1,
    dispatch = all-to-all + the rank's receive-side gather, compute = the GEMMs,
    combine = index_rows + return all-to-all + weighted combine."""
    phases, totals = [], []
    for r in range(len(comp_ms)):
        ph = RankPhases(int((ek["send"] + ALPHA_US / 1e3) * 1e6), int(trans_ms[r] * 1e6),
                        int((disp_a2a + recv_key_fn(r)) * 1e6), int(comp_ms[r] * 1e6),
                        int((ek["back"][r] + comb_a2a + ek["combine"]) * 1e6))
        phases.append(ph)
        totals.append(ph.total(mode, accelerated[r]))
    lat = max(totals)
    return LayerTiming(tuple(phases), tuple(totals), lat, max(p.compute_ns for p in phases),
                       totals.index(lat), mode)


def p2p_layer_timing(comp_ms, trans_ms, accelerated, mode, disp_a2a, comb_a2a, ek):
    """LayerTiming of the host-sync-free peer-memory EP layer (EPMoELayer.forward_device):
    dispatch writes every row straight into its owner's GEMM operand (no receive
    gather), and the down GEMMs store their rows straight into the sources' return
    windows, so the return transfer overlaps the down GEMM (one third of the expert
    flops: 2HI of 6HI per pair). schedule = router/align/pack + C1; dispatch = a2a
    model; compute = GEMMs; combine = the return's excess over the down GEMM +
    combine."""
    phases, totals = [], []
    for r in range(len(comp_ms)):
        ret_exposed = max(0.0, comb_a2a - comp_ms[r] / 3.0)
        ph = RankPhases(int((ek["send"] + ALPHA_US / 1e3) * 1e6), int(trans_ms[r] * 1e6), int(disp_a2a * 1e6),
                        int(comp_ms[r] * 1e6), int((ret_exposed + ek["combine"]) * 1e6))
        phases.append(ph)
        totals.append(ph.total(mode, accelerated[r]))
    lat = max(totals)
    return LayerTiming(tuple(phases), tuple(totals), lat, max(p.compute_ns for p in phases),
                       totals.index(lat), mode)


class VirtualEP:
    """One model shape at EP degree R emulated on cuda:0; weights built once,
    batches (vision fraction, routing skew) regenerated per report."""

    def __init__(self, torch, config: str, R: int, tokens_per_rank: int):
        from . import _lib
        from .workload import make_experts

        self.torch = torch
        self.shape = shape = SHAPES[config]
        E = shape.num_experts
        if E % R:
            raise ValueError(f"{E} experts not divisible by {R}")
        self.R, self.T_local, self.T = R, tokens_per_rank, tokens_per_rank * R
        gu, dn = make_experts(shape)
        self.bias = torch.zeros(E, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
        self.gu, self.dn = gu, dn
        self.epr = E // R
        self.cluster = ClusterConfig(R, 1, self.epr, 1, shape.modality_isolated)
        self.layer = None

    def _layer_for(self, router):
        from .workload import make_shared_expert

        w = MoEWeights.from_hf(self.shape, router, self.gu, self.dn, bias=self.bias,
                               shared=make_shared_expert(self.shape))
        if self.layer is None:
            self.layer = MoELayer(w, max_tokens=self.T, cluster=self.cluster)
        else:
            self.layer.w = w
        return self.layer

    def report(self, vision_frac: float = 0.7, zipf_s: float = 0.57, seed: int = 2024,
               params: RealbParams | None = None) -> dict:
        from .workload import WorkloadSpec, make_batch

        torch, shape, R, T, epr = self.torch, self.shape, self.R, self.T, self.epr
        E, H = shape.num_experts, shape.hidden
        spec = WorkloadSpec(tokens=T, vision_frac=vision_frac, num_ranks=R, zipf_s=zipf_s, seed=seed)
        x, mod, router, _ = make_batch(shape, spec)
        layer = self._layer_for(router)
        params = params or RealbParams()

        # baseline first (bf16 rows of every expert), then realb (NVFP4 rows and weights
        # of its W4A4 experts): both arms' per-rank compute then reads valid operands
        y_base = layer.forward(x, mod, "baseline").y.clone()
        res = layer.forward(x, mod, "realb", params)
        torch.cuda.synchronize()
        accuracy = self.accuracy(x, mod, y_base, res.y, res.plan, layer)
        plan = res.plan
        prec = plan.expert_precision(layer.placement).astype(np.int64)
        vt = res.expert_vt.astype(np.int64)
        rank_vt = vt.reshape(R, epr, 2).sum(1)
        idx = layer.topk_idx[:T].cpu().numpy()

        # every rank's compute under both plans, measured interleaved (clock / power drift
        # hits both arms alike), then the whole one-GPU layer under each strategy
        bf16_ms, realb_ms = measure_rank_compute(torch, layer, T, [np.zeros(E, np.int64), prec], R, epr)
        transform_ms = measure_transform(torch, layer, prec, R, epr)
        whole_realb = _median_ms(torch, lambda: layer.forward(x, mod, "realb", params), reps=5)
        k3_timeline = measure_k3_overlap(torch, layer, x, mod, params)
        whole_bf16 = _median_ms(torch, lambda: layer.forward(x, mod, "baseline"), reps=5)

        # projected full path: engine.py:120-159 overlap rule, measured compute/transform
        pairs = traffic_matrix(idx, self.T_local, epr, R)
        acc = [bool(prec[r * epr] == 1) for r in range(R)]
        disp_bf16, comb = a2a_ms(pairs, np.full(R, 2.0 * H)), a2a_ms(pairs.T.copy(), np.full(R, 2.0 * H))
        disp_fp4 = a2a_ms(pairs, np.where(acc, H / 2 + H / 16, 2.0 * H))
        mode = PipelineMode.OVERLAPPED if plan.active else PipelineMode.SEQUENTIAL
        lt_realb = layer_timing(realb_ms, transform_ms, acc, mode, disp_bf16, comb)
        lt_realb4 = layer_timing(realb_ms, transform_ms, acc, mode, disp_fp4, comb)
        lt_bf16 = layer_timing(bf16_ms, [0.0] * R, [False] * R, PipelineMode.SEQUENTIAL, disp_bf16, comb)
        # with the EP layer's own kernels measured per rank (measure_ep_kernels)
        recv_rows = rank_vt.sum(1)
        ek = measure_ep_kernels(torch, layer, x, mod, self.T_local, recv_rows, acc)
        ep_bf16 = ep_layer_timing(bf16_ms, [0.0] * R, [False] * R, PipelineMode.SEQUENTIAL, disp_bf16, comb, ek,
                                  lambda r: ek["recv_bf16"][r])
        ep_realb = ep_layer_timing(realb_ms, transform_ms, acc, mode, disp_bf16, comb, ek,
                                   lambda r: ek["recv_w4a4"][r] if acc[r] else ek["recv_bf16"][r])
        ep_realb4 = ep_layer_timing(realb_ms, transform_ms, acc, mode, disp_fp4, comb, ek,
                                    lambda r: ek["recv_fp4_packed"][r] if acc[r] else ek["recv_bf16"][r])
        p2p_bf16 = p2p_layer_timing(bf16_ms, [0.0] * R, [False] * R, PipelineMode.SEQUENTIAL, disp_bf16, comb, ek)
        p2p_realb = p2p_layer_timing(realb_ms, transform_ms, acc, mode, disp_fp4, comb, ek)
        text_total = int(rank_vt[:, 1].sum())
        text_fp4 = int(sum(rank_vt[r, 1] for r in range(R) if acc[r]))
        return {
            "what": f"EP{R} emulated on 1 GPU: global batch {T} tokens, plan over {R} virtual ranks, "
                    "per-rank expert compute timed in isolation (layer = max over ranks)",
            "config": shape.name, "ep_ranks": R, "tokens_per_rank": self.T_local,
            "vision_frac": vision_frac, "zipf_s": zipf_s,
            "plan_active": bool(plan.active),
            "plan_w4a4_ranks": sorted(plan.accelerated_ranks), "hot_ranks": sorted(plan.hot_ranks),
            "vision_heavy_ranks": sorted(plan.vision_heavy_ranks),
            "rank_pairs": rank_vt.sum(1).tolist(),
            "device_imbalance": float(rank_vt.sum(1).max() / rank_vt.sum(1).mean()),
            "rank_vision_ratio": [round(float(a / max(1, a + b)), 3) for a, b in rank_vt],
            "text_exposure": text_fp4 / text_total if text_total else 0.0,
            "per_rank_compute_ms": {"bf16": bf16_ms, "realb": realb_ms},
            "transform_ms": transform_ms,
            "compute_only_ms": {"bf16": max(bf16_ms), "realb": max(realb_ms)},
            "compute_only_speedup": max(bf16_ms) / max(realb_ms),
            "one_gpu_whole_layer_ms": {"bf16": whole_bf16, "realb": whole_realb},
            "projected_dispatch_ms": {"bf16_rows": disp_bf16, "fp4_rows_to_w4a4": disp_fp4, "combine": comb},
            "projected_full_path_ms": {"bf16": lt_bf16.layer_latency_ns / 1e6,
                                       "realb": lt_realb.layer_latency_ns / 1e6,
                                       "realb_fp4_dispatch": lt_realb4.layer_latency_ns / 1e6,
                                       "model": f"a2a = {ALPHA_US}us + max_r max(send_r, recv_r) bytes / "
                                                f"{NVLINK_GBPS} GB/s; RankPhases.total overlap rule"},
            "projected_full_path_speedup": lt_bf16.layer_latency_ns / lt_realb.layer_latency_ns,
            "ep_kernels_ms": {k2: v for k2, v in ek.items()},
            "projected_ep_layer_ms": {"bf16": ep_bf16.layer_latency_ns / 1e6,
                                      "realb": ep_realb.layer_latency_ns / 1e6,
                                      "realb_fp4_dispatch": ep_realb4.layer_latency_ns / 1e6,
                                      "model": "RankPhases with the EP layer's measured kernels: schedule = "
                                               "router/align/pack + C1 10us; dispatch = a2a model + receive "
                                               "gather; compute = GEMMs; combine = index_rows + a2a model + "
                                               "combine"},
            "projected_ep_layer_speedup": ep_bf16.layer_latency_ns / ep_realb.layer_latency_ns,
            "projected_ep_layer_speedup_fp4_dispatch": ep_bf16.layer_latency_ns / ep_realb4.layer_latency_ns,
            "projected_full_path_speedup_fp4_dispatch": lt_bf16.layer_latency_ns / lt_realb4.layer_latency_ns,
            "projected_p2p_layer_ms": {"bf16": p2p_bf16.layer_latency_ns / 1e6,
                                       "realb": p2p_realb.layer_latency_ns / 1e6,
                                       "model": "host-sync-free peer-memory layer: direct dispatch into the "
                                                "owners' GEMM operands (NVFP4 to W4A4 ranks, no receive "
                                                "gather); down GEMM stores into the sources' return windows "
                                                "(return overlaps the down GEMM = compute/3); then combine"},
            "projected_p2p_layer_speedup": p2p_bf16.layer_latency_ns / p2p_realb.layer_latency_ns,
            "transform_hidden": all(t <= disp_bf16 for t in transform_ms),
            "k3_overlap_one_gpu": k3_timeline,
            "accuracy": accuracy,
        }

    def accuracy(self, x, mod, y_base, y_realb, plan, layer) -> dict:
        """Per-layer accuracy proxy (the paper's <= 1.2-point downstream delta is not
        reproducible offline): the W4A4 ranks' FP4 weight-error summary
        (quantize_tensor / ErrorSummary, fp4.py:137-170, on the device), the ReaLB
        and FP4-All layer outputs against the all-BF16 layer on the same batch
        (relative RMS, over all / text / vision tokens) and the text exposure
        (metrics.py:72-90)."""
        from .quant import weight_error_summary

        torch, R, epr = self.torch, self.R, self.epr
        I, H = self.shape.intermediate, self.shape.hidden
        vis = mod.bool()
        y_realb = y_realb.clone()  # a view of the layer's output buffer: the next forward reuses it

        def rel(a, b, sel=None):
            if sel is not None:
                a, b = a[sel], b[sel]
            a, b = a.float(), b.float()
            d = float(torch.linalg.vector_norm(b))
            return float(torch.linalg.vector_norm(a - b)) / d if d > 0 else 0.0

        acc_ranks = sorted(plan.accelerated_ranks)
        werr = {}
        for r in acc_ranks:
            e0, e1 = r * epr, (r + 1) * epr
            werr[str(r)] = weight_error_summary([layer.w.w_gu[e0 * 2 * I:e1 * 2 * I], layer.w.w_d[e0 * H:e1 * H]])
        y_fp4 = layer.forward(x, mod, "fp4all", RealbParams(global_batch_threshold=0)).y
        torch.cuda.synchronize()
        return {"fp4_weight_error_w4a4_ranks": werr,
                "realb_vs_bf16_layer_rel": {"all": rel(y_realb, y_base), "text": rel(y_realb, y_base, ~vis),
                                            "vision": rel(y_realb, y_base, vis)},
                "fp4all_vs_bf16_layer_rel": {"all": rel(y_fp4, y_base), "text": rel(y_fp4, y_base, ~vis),
                                             "vision": rel(y_fp4, y_base, vis)},
                "what": "W4A4 ranks' FP4 weight error (device quantize_tensor / ErrorSummary) and layer-output "
                        "deltas vs the all-BF16 layer on the same batch; text exposure is reported beside"}


def virtual_ep_report(args, torch, R: int = 8) -> dict:
    """bench.py's virtual-EP8 block at the bench workload."""
    shape = SHAPES[args.config]
    if shape.num_experts % R:
        return {"skipped": f"{shape.num_experts} experts not divisible by {R}"}
    return VirtualEP(torch, args.config, R, args.tokens).report(args.vision_frac)
