"""One ReaLB MoE layer on one GPU (one EP rank, or all ranks of a 1-GPU run).

This module takes the slot of ``moesim.engine.simulate_layer`` (engine.py:120-159):
instead of evaluating cost formulas it executes the layer with the sm_100a
kernels of the C-ABI library and reports the same per-rank phase schema
(``RankPhases``/``LayerTiming``, engine.py:55-86) filled from CUDA events.

Per layer, all stream-ordered with NO host synchronisation:
  K1+K2 router_topk_stats            main stream   logits, top-k, (v,t) chunk counts
  align_plan                         main stream   expert totals, P1 plan_realb ON THE
                                                   DEVICE (balancers.py:89-122 op order),
                                                   grouped row space per precision
  K3 quantise W4A4 experts' weights  SIDE stream   reads the device plan; overlaps dispatch
  dispatch_permute (+K4 act quant)   main stream
  K5 / K6 grouped GEMMs (+SwiGLU)    main stream   (K6 waits on the side stream)
  combine                            main stream
The plan and counts are copied back asynchronously and exposed lazily on the
returned LayerResult (valid until the next forward() of the same layer).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .policy import ClusterConfig, Precision, PrecisionPlan, RealbParams, place_experts_static


# ----------------------------------------------------------------- shapes
@dataclass(frozen=True)
class MoEShape:
    """MoE-layer shape of a model family (SURVEY.md §8 config shorthand)."""

    name: str
    num_experts: int
    top_k: int
    hidden: int
    intermediate: int
    scoring: int
    routed_scaling: float = 1.0
    norm_min: float = 1e-12
    modality_isolated: bool = False
    # shared-expert MLP intermediate size (moe_intermediate x n_shared_experts; 0: none).
    # Not part of ReaLB's policy (never quantised, not expert-parallel); computed on
    # its own stream, overlapped with the routed path, added in the combine.
    shared_intermediate: int = 0


SHAPES = {
    # 8 experts top-2, H=512 (BASELINE.json configs[0]); I=1024 recorded choice
    "tiny": MoEShape("tiny-mmoe", 8, 2, 512, 1024, _lib.SCORE_SOFTMAX_RENORM),
    # Kimi-VL-A3B (DeepSeek-V3 family router: sigmoid, renorm, x routed_scaling)
    "kimi": MoEShape("kimi-vl-a3b", 64, 6, 2048, 1408, _lib.SCORE_SIGMOID_RENORM, 2.446),
    # the same layer with Kimi-VL's 2 shared experts (DeepSeek-V3 family: one dense
    # MLP of 2 x 1408 on every token, transformers deepseek_v3 DeepseekV3MoE)
    "kimi_shared": MoEShape("kimi-vl-a3b+shared", 64, 6, 2048, 1408, _lib.SCORE_SIGMOID_RENORM, 2.446,
                            shared_intermediate=2816),
    # Qwen3-VL-30B-A3B (softmax, top-k, renorm)
    "qwen": MoEShape("qwen3-vl-30b-a3b", 128, 8, 2048, 768, _lib.SCORE_SOFTMAX_RENORM),
    # ERNIE-4.5-VL-A3B modality-split MoE: vision group (ReaLB applies, isolated)
    "ernie_vision": MoEShape("ernie-4.5-vl-a3b-vision", 64, 6, 2560, 512,
                             _lib.SCORE_SOFTMAX_CLAMPNORM, modality_isolated=True),
    "ernie_text": MoEShape("ernie-4.5-vl-a3b-text", 64, 6, 2560, 1536, _lib.SCORE_SOFTMAX_CLAMPNORM),
}


def host_layout(counts, prec, nchunks: int = 1) -> tuple[np.ndarray, int]:
    """Host construction of the int32 grouped-row layout words realb_moe_align
    builds on the device (include/realb.h) from per-expert row counts and
    precision codes: used to run the grouped GEMMs on an arbitrary (expert ->
    rows) assignment, e.g. an EPLB rank's replica shares. -> (layout, rows used)."""
    counts = np.asarray(counts, np.int64)
    prec = np.asarray(prec, np.int64)
    E = len(counts)
    lay = np.zeros(int(_lib.load().realb_layout_words(E, nchunks)), np.int32)
    padded = (counts + 127) // 128 * 128
    row_start = np.concatenate([[0], np.cumsum(padded)[:-1]])
    lay[8:8 + E] = row_start
    lay[8 + E:8 + 2 * E] = counts
    for p in (0, 1):
        g = np.flatnonzero(prec == p)
        base = 8 + 3 * E + p * (2 * E + 1)
        lay[base:base + len(g)] = g
        mt = padded[g] // 128
        lay[base + E:base + E + len(g) + 1] = np.concatenate([[0], np.cumsum(mt)])
        pbase = 8 + 3 * E + 2 * (2 * E + 1) + p * (E + 1)
        lay[pbase:pbase + len(g) + 1] = np.concatenate([[0], np.cumsum((mt + 1) // 2)])
        lay[1 + p] = len(g)
    lay[0] = int(padded.sum())
    return lay, int(padded.sum())


# ----------------------------------------------------------------- timing schema
class PipelineMode(enum.Enum):
    SEQUENTIAL = "sequential"
    OVERLAPPED = "overlapped"


@dataclass(frozen=True)
class RankPhases:
    """Per-rank phase times in ns (engine.py:55-76), here measured with CUDA events."""

    schedule_ns: int
    transform_ns: int
    dispatch_ns: int
    compute_ns: int
    combine_ns: int

    def total(self, mode: PipelineMode, accelerated: bool) -> int:
        if mode is PipelineMode.OVERLAPPED and accelerated:
            return max(self.dispatch_ns, self.schedule_ns + self.transform_ns) + self.compute_ns + self.combine_ns
        return self.schedule_ns + self.transform_ns + self.dispatch_ns + self.compute_ns + self.combine_ns


@dataclass(frozen=True)
class LayerTiming:
    per_rank: tuple[RankPhases, ...]
    per_rank_total_ns: tuple[int, ...]
    layer_latency_ns: int
    compute_only_ns: int
    critical_rank: int
    pipeline_mode: PipelineMode


# ----------------------------------------------------------------- weights
@dataclass
class MoEWeights:
    """Layer weights on the device in kernel layout.

    router   bf16 [E, H]
    bias     fp32 [E] selection bias (e_score_correction_bias) or None
    w_gu     bf16 [E*2I, H]: per expert, gate/up rows interleaved in 128-row
             halves (block b: gate[128b:128b+128], up[128b:128b+128]) so the
             SwiGLU epilogue sees gate and up of the same outputs in one tile
             (D4)
    w_d      bf16 [E*H, I]
    """

    shape: MoEShape
    router: torch.Tensor
    bias: torch.Tensor | None
    w_gu: torch.Tensor
    w_d: torch.Tensor
    shared_gu: torch.Tensor | None = None  # bf16 [2*Is, H], 128-row gate/up interleave
    shared_d: torch.Tensor | None = None   # bf16 [H, Is]

    @staticmethod
    def interleave_gate_up(gate_up_hf: torch.Tensor) -> torch.Tensor:
        """HF layout gate_up_proj [E, 2I, H] (gate rows first) -> kernel layout [E*2I, H]."""
        E, I2, H = gate_up_hf.shape
        I = I2 // 2
        g = gate_up_hf[:, :I].reshape(E, I // 128, 128, H)
        u = gate_up_hf[:, I:].reshape(E, I // 128, 128, H)
        return torch.stack([g, u], dim=2).reshape(E * I2, H).contiguous()

    @classmethod
    def from_hf(cls, shape: MoEShape, router, gate_up_proj, down_proj, bias=None, device="cuda",
                shared=None):
        """router [E,H], gate_up_proj [E,2I,H], down_proj [E,H,I] (HF conventions);
        shared: (gate_up [2Is,H], down [H,Is]) of the shared-expert MLP, or None."""
        E, H, I = shape.num_experts, shape.hidden, shape.intermediate
        assert tuple(gate_up_proj.shape) == (E, 2 * I, H) and tuple(down_proj.shape) == (E, H, I)
        bf = torch.bfloat16
        sgu = sd = None
        if shape.shared_intermediate:
            if shared is None:
                raise ValueError(f"{shape.name} has a shared expert: pass shared=(gate_up, down)")
            Is = shape.shared_intermediate
            assert tuple(shared[0].shape) == (2 * Is, H) and tuple(shared[1].shape) == (H, Is)
            sgu = cls.interleave_gate_up(shared[0].to(device=device, dtype=bf)[None])
            sd = shared[1].to(device=device, dtype=bf).contiguous()
        return cls(
            shape=shape,
            router=router.to(device=device, dtype=bf).contiguous(),
            bias=None if bias is None else bias.to(device=device, dtype=torch.float32).contiguous(),
            w_gu=cls.interleave_gate_up(gate_up_proj.to(device=device, dtype=bf)),
            w_d=down_proj.to(device=device, dtype=bf).reshape(E * H, I).contiguous(),
            shared_gu=sgu, shared_d=sd,
        )


# ----------------------------------------------------------------- the layer
_STRATEGY_CODE = {"baseline": 0, "eplb": 0, "async-eplb": 0, "fp4all": 1, "realb": 2, "realb-seq": 2}


class LayerResult:
    """Output of one layer call. ``plan`` and ``expert_vt`` are read back lazily
    (an event-guarded pinned copy), so the step itself never synchronises."""

    def __init__(self, y, layer, plan_host, vt_host, event, placement, cluster):
        self.y = y
        self._plan_host, self._vt_host, self._event = plan_host, vt_host, event
        self._placement, self._cluster = placement, cluster
        self._plan = None

    @property
    def expert_vt(self) -> np.ndarray:
        self._event.synchronize()
        return self._vt_host.numpy().copy()

    @property
    def plan(self) -> PrecisionPlan:
        if self._plan is None:
            self._event.synchronize()
            po = self._plan_host.numpy()
            R = self._cluster.num_ranks
            flags = po[3:3 + R]
            active = bool(po[0])
            self._plan = PrecisionPlan(
                tuple(Precision.W4A4 if f & 4 else Precision.W16A16 for f in flags),
                frozenset(int(r) for r in np.flatnonzero(flags & 1)),
                frozenset(int(r) for r in np.flatnonzero(flags & 2)),
                active)
        return self._plan


def operand_noise_(t: torch.Tensor, kind: str = "bf16") -> torch.Tensor:
    """Fill a GEMM operand workspace with in-distribution values, in place.

    Grouped GEMMs multiply every row of a 128-row m-tile, including the padding
    rows at the end of each expert's segment, whose results are never read.
    Those rows keep whatever the buffer held. Measured on B200
    (scripts/bench_k5_data.py), K5 gate_up runs ~13 % slower when the padding
    rows are zero (fresh allocations, memsets) than when they hold activation-like
    values, as they do in steady-state serving, where they keep earlier batches'
    rows. Initialising the workspaces this way gives every batch the
    steady-state behaviour. Results are unaffected: padding rows are never read.
    kind: "bf16" (N(0, 1)), "codes" (uniform E2M1 bytes), "sf" (E4M3 1.0 scales)."""
    flat = t.view(-1)
    step = 1 << 26
    for i in range(0, flat.numel(), step):
        part = flat[i:i + step]
        if kind == "bf16":
            part.normal_()
        elif kind == "codes":
            part.random_(0, 256)
        else:
            part.fill_(0x38)
    return t


class CapturedLayer:
    """A MoE layer forward recorded as a CUDA graph (MoELayer.capture)."""

    def __init__(self, graph, y, layer):
        self.graph, self.y, self.layer = graph, y, layer

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.y


class SharedExpertMLP:
    """The shared-expert MLP (every token; BF16 K5: SwiGLU gate_up, then down) on
    its own stream: start() forks it off the current stream, join() makes the
    current stream wait and returns the bf16 [T, H] output for the combine's
    addend. Used by the single-GPU layer and by every EP rank (the shared expert
    is replicated, not expert-parallel)."""

    def __init__(self, gate_up: torch.Tensor, down: torch.Tensor, max_tokens: int, device):
        self.gu, self.d = gate_up, down
        self.Is, self.H = down.shape[1], down.shape[0]
        self.h = torch.empty(max_tokens, self.Is, dtype=torch.bfloat16, device=device)
        self.y = torch.empty(max_tokens, self.H, dtype=torch.bfloat16, device=device)
        self.stream = torch.cuda.Stream(device=device)
        self.device = device
        self._layouts = {}

    def layout(self, T: int) -> torch.Tensor:
        """One dense group of T rows (cached per T; built before any graph capture,
        the layers run an eager call first)."""
        lay = self._layouts.get(T)
        if lay is None:
            lay = torch.from_numpy(host_layout([T], [0])[0]).to(self.device)
            self._layouts[T] = lay
        return lay

    def start(self, x: torch.Tensor) -> None:
        T = x.shape[0]
        lay = self.layout(T).data_ptr()
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            sp = _lib.stream_ptr(self.stream)
            _lib.call("realb_grouped_gemm_bf16", x.data_ptr(), self.gu.data_ptr(), T, 2 * self.Is, self.H, 1,
                      lay, _lib.PREC_W16A16, _lib.EPI_SWIGLU, self.h.data_ptr(), 0, sp)
            _lib.call("realb_grouped_gemm_bf16", self.h.data_ptr(), self.d.data_ptr(), T, self.H, self.Is, 1,
                      lay, _lib.PREC_W16A16, _lib.EPI_STORE, self.y.data_ptr(), 0, sp)

    def join(self) -> int:
        torch.cuda.current_stream().wait_stream(self.stream)
        return self.y.data_ptr()


class MoELayer:
    """Executes one MoE layer for ``T`` local tokens with preallocated workspaces.

    ``cluster`` describes the EP topology the precision plan is computed over. On
    one GPU ``cluster.num_ranks`` may exceed 1 ("virtual EP": all experts are local,
    the plan is evaluated per group of experts_per_rank experts exactly as the
    reference would for that many ranks); with R = 1 the plan is never active
    (balancers.py:103-104).
    """

    def __init__(self, weights: MoEWeights, max_tokens: int, cluster: ClusterConfig | None = None,
                 device="cuda", quant_max_ctas: int = 0):
        s = weights.shape
        self.w, self.shape = weights, s
        self.E, self.k, self.H, self.I = s.num_experts, s.top_k, s.hidden, s.intermediate
        if self.I % 128 or self.H % 256 or (2 * self.I) % 256:
            raise ValueError("shape must satisfy I % 128 == 0 and H % 256 == 0")
        self.cluster = cluster or ClusterConfig(1, 1, self.E, 1, s.modality_isolated)
        if self.cluster.total_experts != self.E:
            raise ValueError("cluster.total_experts must equal the number of experts")
        self.placement = place_experts_static(self.cluster)
        self.max_tokens = max_tokens
        self.device = torch.device(device)
        self.quant_max_ctas = quant_max_ctas
        E, k, H, I = self.E, self.k, self.H, self.I
        T = max_tokens
        self.nchunks_max = (T + 63) // 64
        self.rows_cap = ((T * k + E * 127) + 127) // 128 * 128
        dev, bf, u8, i32, f32 = self.device, torch.bfloat16, torch.uint8, torch.int32, torch.float32
        self.logits = torch.empty(T, E, dtype=f32, device=dev)
        self.topk_idx = torch.empty(T, k, dtype=i32, device=dev)
        self.topk_w = torch.empty(T, k, dtype=f32, device=dev)
        self.chunk_counts = torch.empty(self.nchunks_max, E, 2, dtype=i32, device=dev)
        self.layout = torch.zeros(int(_lib.load().realb_layout_words(E, self.nchunks_max)), dtype=i32, device=dev)
        self.expert_vt = torch.empty(E, 2, dtype=i32, device=dev)
        self.expert_vt_host = torch.empty(E, 2, dtype=i32, pin_memory=True)
        self.pair_pos = torch.empty(T, k, dtype=i32, device=dev)
        self.prec_dev = torch.zeros(E, dtype=u8, device=dev)
        self.prec_host = torch.zeros(E, dtype=u8, pin_memory=True)
        self.plan_dev = torch.zeros(3 + self.cluster.num_ranks, dtype=i32, device=dev)
        self.plan_host = torch.zeros(3 + self.cluster.num_ranks, dtype=i32, pin_memory=True)
        R = self.rows_cap
        self.a_bf16 = operand_noise_(torch.empty(R, H, dtype=bf, device=dev))
        # How the W16A16 rows reach K5 (scripts/bench_dispatch.py measures all three):
        #   "copy"   realb_dispatch_permute copies them into a_bf16, then K5
        #   "gather" K5 reads them from x through row_src (cp.async loaders)
        #   "copyin" K5's spare warps copy them into a_bf16 while its mainloop runs,
        #            gated per expert (realb_grouped_gemm_bf16_copyin)
        self.dispatch_mode = "copy"
        # rank_partial: combine with the EP rank-partial return's arithmetic (the slots of a
        # W4A4 rank enter as one bf16 partial per (token, rank); ep.py), so
        # the single-GPU layer with the EP cluster reproduces that EP layer bit for bit
        self.rank_partial = False
        self.row_src = torch.zeros(R, dtype=i32, device=dev)
        self.ready = torch.zeros(E, dtype=i32, device=dev)     # copy-in per-expert row counters
        self.copy_err = torch.zeros(1, dtype=i32, device=dev)  # copy-in wait timeout flag
        self._x_src = None  # (x, T) of the last forward: the gather GEMM's A
        self.h_bf16 = torch.empty(R, I, dtype=bf, device=dev)
        self.rows_out = torch.empty(R, H, dtype=bf, device=dev)
        self.flag = torch.zeros(1, dtype=i32, device=dev)
        self.y_buf = torch.empty(T, H, dtype=bf, device=dev)
        self._fp4 = None  # lazily allocated W4A4 workspaces
        self.side = torch.cuda.Stream(device=dev, priority=0)
        self.shared = None
        if s.shared_intermediate:
            if s.shared_intermediate % 128:
                raise ValueError("shared_intermediate must be a multiple of 128")
            self.shared = SharedExpertMLP(weights.shared_gu, weights.shared_d, T, dev)

    # -- W4A4 workspaces (activations + quantised weights of every expert)
    def _fp4_ws(self):
        if self._fp4 is None:
            E, H, I, R = self.E, self.H, self.I, self.rows_cap
            dev, u8 = self.device, torch.uint8
            self._fp4 = dict(
                a_codes=operand_noise_(torch.empty(R, H // 2, dtype=u8, device=dev), "codes"),
                a_sf=operand_noise_(torch.empty(R * H // 16, dtype=u8, device=dev), "sf"),
                h_codes=torch.empty(R, I // 2, dtype=u8, device=dev),
                h_sf=torch.empty(R * I // 16, dtype=u8, device=dev),
                wgu_codes=torch.empty(E * 2 * I, H // 2, dtype=u8, device=dev),
                wgu_sf=torch.empty(E * 2 * I * H // 16, dtype=u8, device=dev),
                wd_codes=torch.empty(E * H, I // 2, dtype=u8, device=dev),
                wd_sf=torch.empty(E * H * I // 16, dtype=u8, device=dev),
            )
        return self._fp4

    def quantize_experts(self, experts, stream=None):
        """K3: quantise the listed experts' BF16 weights into the W4A4 workspace
        (contiguous runs of experts become one launch each)."""
        ws = self._fp4_ws()
        E, H, I = self.E, self.H, self.I
        sp = _lib.stream_ptr(stream)
        runs = []
        for e in sorted(experts):
            if runs and runs[-1][1] == e:
                runs[-1][1] = e + 1
            else:
                runs.append([e, e + 1])
        for lo, hi in runs:
            r0, r1 = lo * 2 * I, hi * 2 * I
            _lib.call("realb_quantize_nvfp4", self.w.w_gu[r0:r1].data_ptr(), _lib.DT_BF16, r1 - r0, H,
                      ws["wgu_codes"][r0:r1].data_ptr(), ws["wgu_sf"][r0 * H // 16:].data_ptr(),
                      _lib.SF_MMA128x4, self.flag.data_ptr(), self.quant_max_ctas, sp)
            d0, d1 = lo * H, hi * H
            _lib.call("realb_quantize_nvfp4", self.w.w_d[d0:d1].data_ptr(), _lib.DT_BF16, d1 - d0, I,
                      ws["wd_codes"][d0:d1].data_ptr(), ws["wd_sf"][d0 * I // 16:].data_ptr(),
                      _lib.SF_MMA128x4, self.flag.data_ptr(), self.quant_max_ctas, sp)

    # -- individual device steps (all on the current stream)
    def route(self, x: torch.Tensor, modality: torch.Tensor):
        T = x.shape[0]
        s = self.shape
        _lib.call("realb_router_topk_stats", x.data_ptr(), self.w.router.data_ptr(),
                  _lib.ptr(self.w.bias), modality.data_ptr(), T, self.H, self.E, self.k, s.scoring,
                  float(s.routed_scaling), float(s.norm_min), self.logits.data_ptr(),
                  self.topk_idx.data_ptr(), self.topk_w.data_ptr(), self.chunk_counts.data_ptr(),
                  _lib.stream_ptr())

    def align(self, T: int, row_align: int = 128):
        _lib.call("realb_moe_align", self.chunk_counts.data_ptr(), (T + 63) // 64, self.E,
                  self.prec_dev.data_ptr(), row_align, self.layout.data_ptr(),
                  self.expert_vt.data_ptr(), _lib.stream_ptr())

    def align_plan(self, T: int, strategy: str, params: RealbParams):
        """Expert totals + the precision plan evaluated on the device (no sync)."""
        c = self.cluster
        _lib.call("realb_moe_align_plan", self.chunk_counts.data_ptr(), (T + 63) // 64, self.E,
                  c.num_ranks, _STRATEGY_CODE[strategy], float(params.capacity_factor),
                  float(params.modality_threshold), int(params.global_batch_threshold),
                  int(bool(c.modality_isolated)), self.prec_dev.data_ptr(), self.plan_dev.data_ptr(),
                  self.layout.data_ptr(), self.expert_vt.data_ptr(), _lib.stream_ptr())

    def forward(self, x: torch.Tensor, modality: torch.Tensor, strategy: str = "realb",
                params: RealbParams | None = None, out: torch.Tensor | None = None,
                timer=None) -> LayerResult:
        """One MoE layer over the local tokens; stream-ordered, no host sync.

        strategy "baseline" (and the EPLB tags) runs the all-BF16 comparator with
        exactly the same kernels minus the NVFP4 ones; "realb"/"fp4all" evaluate
        the plan on the device and launch the W4A4 machinery (K3 on the side
        stream, K4 in dispatch, K6), which is a no-op for experts the plan keeps
        at W16A16."""
        if strategy not in _STRATEGY_CODE:
            raise ValueError(f"unknown strategy {strategy!r}")
        params = params or RealbParams()
        T = x.shape[0]
        if T > self.max_tokens:
            raise ValueError("more tokens than the layer was sized for")
        E, k, H, I = self.E, self.k, self.H, self.I
        nch = (T + 63) // 64
        main = torch.cuda.current_stream()
        sp = _lib.stream_ptr(main)
        shared = self.shared is not None and T > 0
        mark = timer.mark if timer is not None else (lambda *a, **kw: None)
        if shared:  # overlapped with the whole routed path, joined before the combine
            self.shared.start(x)
        mark("route_start", main)
        self.route(x, modality)
        self.align_plan(T, strategy, params)
        mark("plan_end", main)
        # NVFP4 launches are needed unless the plan provably stays all-W16A16: the
        # baseline strategies, or realb on one rank with C >= 1 (a rank's load is
        # then exactly the mean, never > C x mean; balancers.py:103-104). This is a
        # static property of (strategy, R, C), not of the data.
        code = _STRATEGY_CODE[strategy]
        mixed = code == 1 or (code == 2 and not (self.cluster.num_ranks == 1
                                                 and params.capacity_factor >= 1.0))
        # realb-seq: the reference's sequential ablation (engine.py:162-167): K3 on the
        # main stream, so the transform is NOT hidden behind dispatch
        k3_stream = main if strategy == "realb-seq" else self.side
        if mixed:
            ws = self._fp4_ws()
            if k3_stream is not main:
                self.side.wait_stream(main)
            with torch.cuda.stream(k3_stream):
                ssp = _lib.stream_ptr(k3_stream)
                mark("k3_start", k3_stream)
                # gate_up and down weights of the W4A4 experts in one launch
                _lib.call("realb_quantize_experts2_nvfp4",
                          self.w.w_gu.data_ptr(), 2 * I, H, ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(),
                          self.w.w_d.data_ptr(), H, I, ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(),
                          E, self.prec_dev.data_ptr(), self.flag.data_ptr(), self.quant_max_ctas, ssp)
                mark("k3_end", k3_stream)
        else:
            ws = None
        mark("dispatch_start", main)
        self._x_src = (x, T)
        if self.dispatch_mode in ("gather", "copyin"):
            _lib.call("realb_dispatch_index", x.data_ptr(), self.topk_idx.data_ptr(), T, H, E, k,
                      self.prec_dev.data_ptr(), self.layout.data_ptr(), nch, self.rows_cap,
                      self.pair_pos.data_ptr(), self.row_src.data_ptr(),
                      _lib.ptr(ws["a_codes"]) if ws else None, _lib.ptr(ws["a_sf"]) if ws else None,
                      self.flag.data_ptr(), sp)
        else:
            _lib.call("realb_dispatch_permute", x.data_ptr(), self.topk_idx.data_ptr(), T, H, E, k,
                      self.prec_dev.data_ptr(), self.layout.data_ptr(), nch, self.rows_cap,
                      self.pair_pos.data_ptr(), self.a_bf16.data_ptr(),
                      _lib.ptr(ws["a_codes"]) if ws else None, _lib.ptr(ws["a_sf"]) if ws else None,
                      self.flag.data_ptr(), sp)
        mark("dispatch_end", main)
        lay = self.layout.data_ptr()
        mark("gate_up_start", main)
        self._gate_up_bf16(lay, sp, in_forward=True)
        mark("gate_up_end", main)
        if ws is not None:
            mark("fp4_ready", main)  # main stream reaches the first W4A4 GEMM
            if k3_stream is not main:
                main.wait_stream(self.side)
            mark("fp4_start", main)
            _lib.call("realb_grouped_gemm_nvfp4", ws["a_codes"].data_ptr(), ws["a_sf"].data_ptr(),
                      ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(), self.rows_cap, 2 * I, H, E,
                      lay, _lib.EPI_SWIGLU, None, ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(), 0, sp)
        mark("down_start", main)
        _lib.call("realb_grouped_gemm_bf16", self.h_bf16.data_ptr(), self.w.w_d.data_ptr(),
                  self.rows_cap, H, I, E, lay, _lib.PREC_W16A16, _lib.EPI_STORE,
                  self.rows_out.data_ptr(), 0, sp)
        if ws is not None:
            _lib.call("realb_grouped_gemm_nvfp4", ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(),
                      ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(), self.rows_cap, H, I, E, lay,
                      _lib.EPI_STORE, self.rows_out.data_ptr(), None, None, 0, sp)
        mark("down_end", main)
        y = self.y_buf[:T] if out is None else out
        addend = self.shared.join() if shared else None
        if self.rank_partial:  # the EP rank-partial return's numerics (W4A4 ranks' slots pre-summed)
            _lib.call("realb_combine_partial", self.rows_out.data_ptr(), self.pair_pos.data_ptr(),
                      self.topk_w.data_ptr(), self.topk_idx.data_ptr(), self.prec_dev.data_ptr(),
                      self.cluster.experts_per_rank, T, H, k, addend, -1, 0, y.data_ptr(), sp)
        else:
            _lib.call("realb_combine", self.rows_out.data_ptr(), self.pair_pos.data_ptr(),
                      self.topk_w.data_ptr(), T, H, k, addend, y.data_ptr(), sp)
        mark("combine_end", main)
        if torch.cuda.is_current_stream_capturing():
            return LayerResult(y, self, self.plan_host, self.expert_vt_host, None, self.placement,
                               self.cluster)
        # lazy, asynchronous read-back of the plan and the counts (pinned, event-guarded)
        self.plan_host.copy_(self.plan_dev, non_blocking=True)
        self.expert_vt_host.copy_(self.expert_vt, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(main)
        return LayerResult(y, self, self.plan_host, self.expert_vt_host, ev, self.placement, self.cluster)

    def capture(self, x: torch.Tensor, modality: torch.Tensor, strategy: str = "realb",
                params: RealbParams | None = None, out: torch.Tensor | None = None,
                timer=None) -> "CapturedLayer":
        """Record one forward() into a CUDA graph over the given (static) input
        tensors. The forward is host-sync-free, so the whole layer — router,
        device-side plan, side-stream K3, dispatch, both GEMM precisions, combine
        — replays as one graph launch. Refill ``x``/``modality`` in place and call
        ``replay()``; the output is ``captured.y``."""
        self.forward(x, modality, strategy, params, out)  # warm-up: allocations, kernel attributes
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            # a timer's events must be external (event-record nodes) to time replays
            res = self.forward(x, modality, strategy, params, out, timer=timer)
        return CapturedLayer(g, res.y, self)

    def expert_compute(self, T: int, prec: np.ndarray) -> None:
        """Re-run only the expert GEMMs of the experts whose code in ``prec`` is
        0 (W16A16) or 1 (W4A4); code 2 excludes an expert. Operates on the rows the
        last forward() dispatched (the codes of included experts must match it).
        Used to time one (virtual) EP rank's compute in isolation."""
        E, H, I = self.E, self.H, self.I
        self.prec_host.numpy()[:] = prec
        self.prec_dev.copy_(self.prec_host, non_blocking=True)
        self.align(T)
        sp, lay = _lib.stream_ptr(), self.layout.data_ptr()
        if (prec == 0).any():
            self._gate_up_bf16(lay, sp)
            _lib.call("realb_grouped_gemm_bf16", self.h_bf16.data_ptr(), self.w.w_d.data_ptr(),
                      self.rows_cap, H, I, E, lay, _lib.PREC_W16A16, _lib.EPI_STORE,
                      self.rows_out.data_ptr(), 0, sp)
        if (prec == 1).any():
            ws = self._fp4_ws()
            _lib.call("realb_grouped_gemm_nvfp4", ws["a_codes"].data_ptr(), ws["a_sf"].data_ptr(),
                      ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(), self.rows_cap, 2 * I, H, E,
                      lay, _lib.EPI_SWIGLU, None, ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(), 0, sp)
            _lib.call("realb_grouped_gemm_nvfp4", ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(),
                      ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(), self.rows_cap, H, I, E, lay,
                      _lib.EPI_STORE, self.rows_out.data_ptr(), None, None, 0, sp)

    def bf16_compute_on(self, layout_dev: torch.Tensor) -> None:
        """The BF16 expert GEMMs (gate_up + SwiGLU, down) over an explicit layout
        (host_layout): times an arbitrary per-expert row assignment (an EPLB
        rank's hosted replicas) on this layer's weights; reads whatever rows the
        activation buffers hold."""
        E, H, I = self.E, self.H, self.I
        sp, lay = _lib.stream_ptr(), layout_dev.data_ptr()
        self._gate_up_bf16(lay, sp)
        _lib.call("realb_grouped_gemm_bf16", self.h_bf16.data_ptr(), self.w.w_d.data_ptr(),
                  self.rows_cap, H, I, E, lay, _lib.PREC_W16A16, _lib.EPI_STORE,
                  self.rows_out.data_ptr(), 0, sp)

    def _gate_up_bf16(self, lay: int, sp: int, in_forward: bool = False) -> None:
        """K5 gate_up (+ SwiGLU) of the W16A16 experts: the gather form reads the
        rows of the last forward's x through row_src; the copy form reads a_bf16;
        the copy-in form (forward only) fills a_bf16 inside the GEMM."""
        H, I, E = self.H, self.I, self.E
        if self.dispatch_mode == "copyin" and in_forward:
            x, T = self._x_src
            _lib.call("realb_grouped_gemm_bf16_copyin", x.data_ptr(), self.row_src.data_ptr(),
                      self.a_bf16.data_ptr(), self.w.w_gu.data_ptr(), self.rows_cap, 2 * I, H, E, lay,
                      _lib.PREC_W16A16, _lib.EPI_SWIGLU, self.h_bf16.data_ptr(), self.ready.data_ptr(),
                      self.copy_err.data_ptr(), 0, sp)
        elif self.dispatch_mode == "gather" and self._x_src is not None:
            x, T = self._x_src
            if T == 0:
                return
            _lib.call("realb_grouped_gemm_bf16_gather", x.data_ptr(), T, self.row_src.data_ptr(),
                      self.w.w_gu.data_ptr(), self.rows_cap, 2 * I, H, E, lay, _lib.PREC_W16A16,
                      _lib.EPI_SWIGLU, self.h_bf16.data_ptr(), 0, sp)
        else:
            _lib.call("realb_grouped_gemm_bf16", self.a_bf16.data_ptr(), self.w.w_gu.data_ptr(),
                      self.rows_cap, 2 * I, H, E, lay, _lib.PREC_W16A16, _lib.EPI_SWIGLU,
                      self.h_bf16.data_ptr(), 0, sp)

    def check_flag(self):
        from .quant import QuantizationDomainError

        if int(self.copy_err.item()):
            self.copy_err.zero_()
            raise RuntimeError("copy-in dispatch: a K5 producer timed out waiting for its rows")
        if int(self.flag.item()):
            self.flag.zero_()
            raise QuantizationDomainError("non-finite value reached the NVFP4 quantiser")


class ModalitySplitMoELayer:
    """A modality-split MoE layer (ERNIE-4.5-VL: separate text and vision expert
    groups; BASELINE configs[3]). Text tokens go through the text group at
    W16A16; vision tokens through the vision group, where ReaLB applies with the
    modality-isolated policy (every loaded hot rank is eligible,
    balancers.py:105-106). The split is boolean-mask indexing on the token-type
    mask — the surrounding model does the same (a host sync, as there) — and the
    two groups' outputs are scattered back into token order."""

    def __init__(self, text: MoELayer, vision: MoELayer):
        if not vision.cluster.modality_isolated:
            raise ValueError("the vision group must use a modality_isolated cluster")
        self.text, self.vision = text, vision

    def forward(self, x: torch.Tensor, modality: torch.Tensor, strategy: str = "realb",
                params: RealbParams | None = None, out: torch.Tensor | None = None):
        """-> (y [T, H] bf16, text LayerResult or None, vision LayerResult or None)"""
        vis = modality.bool()
        iv = vis.nonzero().squeeze(1)
        it = (~vis).nonzero().squeeze(1)
        y = torch.empty_like(x) if out is None else out
        rt = rv = None
        if it.numel():
            rt = self.text.forward(x.index_select(0, it), modality.index_select(0, it), "baseline")
            y.index_copy_(0, it, rt.y)
        if iv.numel():
            rv = self.vision.forward(x.index_select(0, iv), modality.index_select(0, iv), strategy, params)
            y.index_copy_(0, iv, rv.y)
        return y, rt, rv
