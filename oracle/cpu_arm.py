"""CPU arm of bench.py — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

The reference's CPU implementation of the MoE-layer path, as the oracle
restates it, run on the host cores: bench.py's ``cpu_baseline`` leg and its
``--impl reference`` arm execute this module and nothing from the product
package (no paper_2604_19503_b200 import, no librealb_b200.so), so the only
native code they load is oracle/build/liboracle_fp4.so.

One step = one MoE layer over a batch of synthetic multimodal tokens of the
named shape (the workload model of paper_2604_19503_b200/workload.py, restated
here in numpy: Zipf popularity with the hot rank's experts on the most popular
slots and modality affinity, tracegen.py:37-48/:114-133/:164-184; tokens built
with margins over unit router rows so the router selects the planned set):

  route            oracle/moe_ref.route (fp32 logits, stable top-k, family weights)
  stats            per-expert (vision, text) pair counts
  policy           oracle/policy_ref: aggregate_rank_loads (core.py:106-130) +
                   plan_for / plan_realb (balancers.py:89-122, :202-219)
  experts          oracle/moe_ref.moe_layer: fp32 GEMMs (numpy BLAS, all host
                   threads), W4A4 experts through the reference block rule
  combine          fp32 weighted top-k sum, one bf16 rounding

Also timed: the reference quantiser rule (oracle/fp4_numpy,
float64 numpy = moesim.fp4.quantize_blocks' algorithm, 1 core), the C
quantiser port, and the reference policy per layer.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import moe_ref, policy_ref

# (E, k, H, I, scoring, routed_scaling, modality_isolated)  -- DESIGN.md §5 / SURVEY §8 shapes
SHAPES = {
    "tiny": (8, 2, 512, 1024, moe_ref.SOFTMAX_RENORM, 1.0, False),
    "kimi": (64, 6, 2048, 1408, moe_ref.SIGMOID_RENORM, 2.446, False),
    "kimi_shared": (64, 6, 2048, 1408, moe_ref.SIGMOID_RENORM, 2.446, False),
    "qwen": (128, 8, 2048, 768, moe_ref.SOFTMAX_RENORM, 1.0, False),
    "ernie_vision": (64, 6, 2560, 512, moe_ref.SOFTMAX_CLAMPNORM, 1.0, True),
}
NAMES = {"tiny": "tiny-mmoe", "kimi": "kimi-vl-a3b", "kimi_shared": "kimi-vl-a3b+shared",
         "qwen": "qwen3-vl-30b-a3b", "ernie_vision": "ernie-4.5-vl-a3b-vision"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _bf16(a: np.ndarray) -> np.ndarray:
    """float32 -> bf16 values (RNE), in place (finite inputs of moderate size)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = a.view(np.uint32)
    b += np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    b &= np.uint32(0xFFFF0000)
    return a


class CpuLayerArm:
    def __init__(self, config: str, tokens: int, vision_frac: float = 0.7, num_ranks: int = 1,
                 seed: int = 2024, threads: int | None = None):
        E, k, H, I, scoring, scaling, iso = SHAPES[config]
        self.config, self.E, self.k, self.H, self.I = config, E, k, H, I
        self.scoring, self.scaling, self.iso = scoring, scaling, iso
        self.R = num_ranks if E % max(1, num_ranks) == 0 else 1
        self.T = tokens
        self.threads = threads or os.cpu_count() or 1
        self._limit = None
        try:  # numpy BLAS on every host thread
            from threadpoolctl import threadpool_limits

            self._limit = threadpool_limits(self.threads)
        except Exception:  # noqa: BLE001
            pass
        rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(77,)))
        # router: unit rows x gain 0.25, bf16
        unit = rng.standard_normal((E, H), dtype=np.float32)
        unit /= np.linalg.norm(unit, axis=1, keepdims=True)
        self.router = _bf16(unit * 0.25)
        # routing model (numpy restatement of workload.sample_routing)
        epr = E // 8 if E % 8 == 0 else E
        hot = int(rng.integers(max(1, E // epr)))
        slots = np.arange(1, E + 1, dtype=np.float64) ** -0.57 * np.exp(0.3 * rng.standard_normal(E))
        top = rng.permutation(np.arange(hot * epr, (hot + 1) * epr))[:max(1, epr // 2)]
        order = np.concatenate([top, rng.permutation(np.setdiff1d(np.arange(E), top))])
        pop = np.zeros(E)
        pop[order] = slots
        pop /= pop.sum()
        f = np.full(E, 0.31)
        f[hot * epr:(hot + 1) * epr] = 0.93
        n_vis = int(round(tokens * vision_frac))
        self.mod = np.zeros(tokens, np.uint8)
        self.mod[rng.permutation(tokens)[:n_vis]] = 1
        lv, lt = np.log(pop * f + 1e-300), np.log(pop * (1 - f) + 1e-300)
        if iso:
            lt = lv
        keys = np.where(self.mod[:, None] == 1, lv, lt) + rng.gumbel(size=(tokens, E))
        planned = np.argsort(-keys, axis=1, kind="stable")[:, :k]
        amp = np.zeros((tokens, E), np.float32)
        np.put_along_axis(amp, planned, (np.float32(12.0) - np.arange(k, dtype=np.float32)) / np.float32(0.25),
                          axis=1)
        self.x = _bf16(rng.standard_normal((tokens, H), dtype=np.float32) + amp @ unit)
        # experts N(0, 0.02), bf16, HF layout, generated expert by expert
        self.gate_up = np.empty((E, 2 * I, H), np.float32)
        self.down = np.empty((E, H, I), np.float32)
        for e in range(E):
            self.gate_up[e] = _bf16(rng.standard_normal((2 * I, H), dtype=np.float32) * np.float32(0.02))
            self.down[e] = _bf16(rng.standard_normal((H, I), dtype=np.float32) * np.float32(0.02))
        self.assignment = tuple((e // (E // self.R),) for e in range(E))

    # ------------------------------------------------------------ one layer step
    def plan(self, vt: np.ndarray):
        loads = policy_ref.aggregate_rank_loads({e: (int(vt[e, 0]), int(vt[e, 1])) for e in range(self.E)
                                                 if vt[e].any()}, self.assignment, self.R)
        return policy_ref.plan_for("realb", loads, isolated=self.iso)

    def step(self) -> float:
        t0 = time.perf_counter()
        logits, idx, _ = moe_ref.route(self.x, self.router, self.k, self.scoring, routed_scaling=self.scaling)
        vt = moe_ref.expert_counts(idx, self.mod, self.E)
        p = self.plan(vt)
        prec = np.array([p["precision"][h[0]] for h in self.assignment], np.int64)
        moe_ref.moe_layer(self.x, self.mod, self.router, self.gate_up, self.down, self.k, self.scoring,
                          expert_prec=prec, routed_scaling=self.scaling, logits=logits)
        return time.perf_counter() - t0

    # ------------------------------------------------------------ BASELINE.md §3 pieces
    def quantiser_rates(self, max_seconds: float = 3.0) -> dict:
        """MB/s of bf16 input: the reference rule in float64 numpy (1 core) and the
        C port, on expert 0's gate_up weights (a bounded sample of one rank-layer)."""
        from . import fp4_numpy, quantize_bf16

        w = self.gate_up[0]
        nbytes_bf16 = w.size * 2
        t = time.perf_counter()
        fp4_numpy.quantize_blocks(w.reshape(-1, 16).astype(np.float64))
        ref_s = time.perf_counter() - t
        bits = (w.view(np.uint32) >> 16).astype(np.uint16)
        t = time.perf_counter()
        quantize_bf16(bits)
        port_s = time.perf_counter() - t
        return {"reference_rule_numpy_MBps": nbytes_bf16 / ref_s / 1e6, "c_port_MBps": nbytes_bf16 / port_s / 1e6,
                "sample": f"expert 0 gate_up of {NAMES[self.config]} ({w.size} bf16 weights, {nbytes_bf16 / 1e6:.1f} MB)",
                "cores": 1}

    def policy_us_per_layer(self, reps: int = 2000) -> dict:
        rng = np.random.default_rng(3)
        vts = [rng.integers(0, 1000, (self.E, 2)) for _ in range(16)]
        t = time.perf_counter()
        for i in range(reps):
            self.plan(vts[i % 16])
        us = (time.perf_counter() - t) / reps * 1e6
        return {"us_per_layer": us, "what": f"aggregate_rank_loads + plan_realb, E={self.E}, R={self.R}",
                "cores": 1}

    def blas_threads(self) -> int:
        try:
            from threadpoolctl import threadpool_info

            return max((int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas"),
                       default=self.threads)
        except Exception:  # noqa: BLE001
            return self.threads

    def describe(self, value: float, kind: str = "port") -> dict:
        self.threads = self.blas_threads()
        return {"value": value, "unit": "tokens/s", "cores": self.threads, "kind": kind,
                "sample": f"{self.T} tokens of the {NAMES[self.config]} workload per step through the full CPU "
                          f"oracle layer (numpy fp32 GEMMs on {self.threads} BLAS threads), plan over R={self.R}",
                "cpu_model": cpu_model(), "host_threads": os.cpu_count()}
