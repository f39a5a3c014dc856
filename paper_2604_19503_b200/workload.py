"""Synthetic multimodal MoE-layer inputs of the named shapes (no checkpoints or
datasets exist offline; BASELINE.json asks for synthetic batches and random-init
weights).

Routing skew follows the reference trace generator's model
(moesim/tracegen.py:35-48, :114-133, :164-184): Zipf(s) popularity over
popularity slots, the hot rank's top half of experts taking the most popular
slots, log-normal jitter per layer, and modality affinity (vision share 0.93 on
hot-rank experts, 0.31 elsewhere). Each token's k experts are drawn from that
model (Gumbel top-k, without replacement) and the hidden state is built as
``h = noise + sum_j a_j * w_hat[e_j]`` with descending margins a_j over unit
router rows, so the real router — GPU or CPU — selects exactly the planned set
(margins >> fp32 rounding).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .moe import MoEShape


@dataclass(frozen=True)
class WorkloadSpec:
    tokens: int
    vision_frac: float = 0.7
    num_ranks: int = 8            # EP ranks the hot-rank model is laid over
    zipf_s: float = 0.57          # tracegen.py:39-41
    hot_rank_vision_frac: float = 0.93
    base_vision_frac: float = 0.31
    popularity_jitter_sigma: float = 0.30
    seed: int = 2024              # the reference default seed (conftest.py:34)
    layer: int = 0
    rank: int = 0                 # DP rank whose local tokens these are
    noise_std: float = 1.0
    margin_top: float = 12.0      # a_0 (selected-expert projection), post-gain
    margin_step: float = 1.0      # a_j = margin_top - j * margin_step
    router_gain: float = 0.25


def expert_popularity(E: int, spec: WorkloadSpec) -> tuple[np.ndarray, int]:
    """Per-expert popularity (sums to 1) and the hot rank for this layer."""
    epr = E // spec.num_ranks
    rng = np.random.default_rng(np.random.SeedSequence(spec.seed, spawn_key=(0, 0)))
    hot = int(rng.integers(spec.num_ranks))
    hot_experts = np.arange(hot * epr, (hot + 1) * epr)
    n_top = max(1, epr // 2)
    top = rng.permutation(hot_experts)[:n_top]
    rest = np.setdiff1d(np.arange(E), top)
    slot_to_expert = np.concatenate([top, rng.permutation(rest)])
    slot_w = np.arange(1, E + 1, dtype=np.float64) ** (-spec.zipf_s)
    lrng = np.random.default_rng(np.random.SeedSequence(spec.seed, spawn_key=(1, spec.layer)))
    if spec.popularity_jitter_sigma > 0:
        slot_w = slot_w * np.exp(spec.popularity_jitter_sigma * lrng.standard_normal(E))
    pop = np.zeros(E)
    pop[slot_to_expert] = slot_w
    return pop / pop.sum(), hot


def sample_routing(shape: MoEShape, spec: WorkloadSpec):
    """modality [T] uint8 and planned expert ids [T, k] (numpy)."""
    E, k, T = shape.num_experts, shape.top_k, spec.tokens
    pop, hot = expert_popularity(E, spec)
    epr = E // spec.num_ranks
    rng = np.random.default_rng(np.random.SeedSequence(spec.seed, spawn_key=(3, spec.layer, spec.rank)))
    n_vis = int(round(T * spec.vision_frac))
    modality = np.zeros(T, np.uint8)
    modality[rng.permutation(T)[:n_vis]] = 1
    f = np.full(E, spec.base_vision_frac)
    f[hot * epr:(hot + 1) * epr] = spec.hot_rank_vision_frac
    logw_v = np.log(pop * f + 1e-300)
    logw_t = np.log(pop * (1 - f) + 1e-300)
    if shape.modality_isolated:  # the vision group serves vision tokens only
        logw_t = logw_v
    g = rng.gumbel(size=(T, E))
    keys = np.where(modality[:, None] == 1, logw_v[None, :], logw_t[None, :]) + g
    idx = np.argsort(-keys, axis=1, kind="stable")[:, :k].astype(np.int32)
    return modality, idx, hot


def make_router(shape: MoEShape, spec: WorkloadSpec, device="cuda") -> tuple[torch.Tensor, torch.Tensor]:
    """Unit router rows (fp32) and the bf16 router weight (unit rows x gain)."""
    gen = torch.Generator(device="cpu").manual_seed(spec.seed * 1009 + 7)
    w = torch.randn(shape.num_experts, shape.hidden, generator=gen, dtype=torch.float32)
    w = w / w.norm(dim=1, keepdim=True)
    return w.to(device), (w * spec.router_gain).to(device=device, dtype=torch.bfloat16)


def make_hidden(shape: MoEShape, spec: WorkloadSpec, unit_router: torch.Tensor, idx: np.ndarray):
    """bf16 [T, H] hidden states whose router logits select ``idx`` with margins."""
    T, k, E = spec.tokens, shape.top_k, shape.num_experts
    dev = unit_router.device
    gen = torch.Generator(device=dev).manual_seed(spec.seed * 31 + spec.layer * 7 + spec.rank)
    x = torch.randn(T, shape.hidden, generator=gen, device=dev) * spec.noise_std
    # add a_j / gain along each selected unit row: logit_e ~ a_j + gain * N(0, 1)
    amp = torch.zeros(T, E, device=dev)
    a = torch.tensor([spec.margin_top - j * spec.margin_step for j in range(k)], device=dev) / spec.router_gain
    amp.scatter_(1, torch.from_numpy(idx).long().to(dev), a.expand(T, k).contiguous())
    x = x + amp @ unit_router
    return x.to(torch.bfloat16)


def make_experts(shape: MoEShape, seed: int = 2024, std: float = 0.02, device="cuda"):
    """HF-layout random-init expert weights N(0, std) (initializer_range
    convention): gate_up_proj [E, 2I, H], down_proj [E, H, I], bf16."""
    E, H, I = shape.num_experts, shape.hidden, shape.intermediate
    gen = torch.Generator(device=device).manual_seed(seed * 17 + 3)
    gu = (torch.randn(E, 2 * I, H, generator=gen, device=device) * std).to(torch.bfloat16)
    dn = (torch.randn(E, H, I, generator=gen, device=device) * std).to(torch.bfloat16)
    return gu, dn


def make_shared_expert(shape: MoEShape, seed: int = 2024, std: float = 0.02, device="cuda"):
    """Random-init shared-expert MLP (HF layout): gate_up [2Is, H] (gate rows first),
    down [H, Is], bf16 N(0, std); None when the shape has no shared expert."""
    Is, H = shape.shared_intermediate, shape.hidden
    if not Is:
        return None
    gen = torch.Generator(device=device).manual_seed(seed * 29 + 11)
    gu = (torch.randn(2 * Is, H, generator=gen, device=device) * std).to(torch.bfloat16)
    dn = (torch.randn(H, Is, generator=gen, device=device) * std).to(torch.bfloat16)
    return gu, dn


def make_batch(shape: MoEShape, spec: WorkloadSpec, device="cuda"):
    """Everything one layer invocation needs: (x bf16 [T,H], modality u8 [T],
    router bf16 [E,H], planned idx [T,k] numpy)."""
    modality, idx, _ = sample_routing(shape, spec)
    unit, router = make_router(shape, spec, device)
    x = make_hidden(shape, spec, unit, idx)
    return x, torch.from_numpy(modality).to(device), router, idx


def make_split_batch(text_shape: MoEShape, vision_shape: MoEShape, spec: WorkloadSpec, device="cuda"):
    """A modality-split (ERNIE) batch: vision tokens routed with margins over the
    vision group's router, text tokens over the text group's (separate router
    seeds), interleaved by a seeded token-type mask. -> (x, modality, router_text,
    router_vision, planned_text, planned_vision)."""
    from dataclasses import replace

    T = spec.tokens
    n_vis = int(round(T * spec.vision_frac))
    rng = np.random.default_rng(np.random.SeedSequence(spec.seed, spawn_key=(4, spec.layer, spec.rank)))
    modality = np.zeros(T, np.uint8)
    modality[rng.permutation(T)[:n_vis]] = 1
    xt, _, rt, pt = make_batch(text_shape, replace(spec, tokens=T - n_vis, vision_frac=0.0), device)
    xv, _, rv, pv = make_batch(vision_shape, replace(spec, tokens=n_vis, vision_frac=1.0, seed=spec.seed + 1),
                               device)
    x = torch.empty(T, text_shape.hidden, dtype=torch.bfloat16, device=device)
    mod = torch.from_numpy(modality).to(device)
    vis = mod.bool()
    x[~vis] = xt
    x[vis] = xv
    return x, mod, rt, rv, pt, pv
