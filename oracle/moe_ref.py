"""CPU ORACLE of the MoE-layer path — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

numpy restatement, step by step, of what one ReaLB MoE layer computes. The
reference (moesim) pins only the policy and the quantiser; everything else is
"parity unpinned" by the reference and defined here:

  router      logits = x . Wg^T in fp32; selection on s = logits + bias, stable
              top-k (descending, ties -> lowest expert id: the convention of
              balancers.py:161-165); weights per family (D1):
                softmax_renorm   p = softmax(l); w = p_sel / sum(p_sel)
                sigmoid_renorm   p = sigmoid(l); w = p_sel / sum(p_sel) * scaling
                softmax_clamp    p = softmax(l); w = p_sel / max(sum(p_sel), norm_min)
  stats       per-expert (vision, text) pair counts -> aggregate_rank_loads
              (core.py:106-130) -> plan_realb (balancers.py:89-122)
  experts     W16A16: g,u = x.Wg^T, x.Wu^T (fp32 acc over bf16 values);
                      h = bf16(silu(g) * u); y = bf16(h . Wd^T)
              W4A4:   same with x, W and h replaced by their reference-block-rule
                      fake-quantised values (fp4.py:108-122, along K, D3)
  combine     out[t] = bf16( sum_j w[t,j] * y[t,j] )  (fp32 accumulate); with the
              rank-partial return (partial_el = experts per rank), the slots of a W4A4
              owner rank enter as one bf16-rounded partial sum per (token, rank)
"""

from __future__ import annotations

import numpy as np

from . import fake_quant

SOFTMAX_RENORM, SIGMOID_RENORM, SOFTMAX_CLAMPNORM = 0, 1, 2


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (RNE) and back to float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = a.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return (b.astype(np.uint32) << 16).view(np.float32)


def topk_stable(scores: np.ndarray, k: int) -> np.ndarray:
    """[T, E] -> [T, k] ids, descending score, ties to the lowest id."""
    order = np.argsort(-scores, axis=1, kind="stable")
    return order[:, :k].astype(np.int32)


def route(x, wg, k, scoring, bias=None, routed_scaling=1.0, norm_min=1e-12, logits=None):
    """x [T,H] float32 (bf16 values), wg [E,H]. ``logits`` may be supplied (the D1
    contract: selection on the device-written logits)."""
    if logits is None:
        logits = x.astype(np.float32) @ wg.astype(np.float32).T
    logits = logits.astype(np.float32)
    s = logits + (bias.astype(np.float32) if bias is not None else 0.0)
    idx = topk_stable(s, k)
    sel = np.take_along_axis(logits, idx, axis=1).astype(np.float64)
    if scoring == SIGMOID_RENORM:
        p = 1.0 / (1.0 + np.exp(-sel))
        w = p / p.sum(axis=1, keepdims=True) * routed_scaling
    else:
        l64 = logits.astype(np.float64)
        m = l64.max(axis=1, keepdims=True)
        z = np.exp(l64 - m).sum(axis=1, keepdims=True)
        p = np.exp(sel - m) / z
        den = p.sum(axis=1, keepdims=True)
        w = p / den if scoring == SOFTMAX_RENORM else p / np.maximum(den, norm_min)
    return logits, idx, w.astype(np.float32)


def expert_counts(idx: np.ndarray, modality: np.ndarray, E: int) -> np.ndarray:
    """[E, 2] (vision, text) pair counts."""
    vt = np.zeros((E, 2), np.int64)
    vis = np.repeat(modality.astype(bool), idx.shape[1])
    np.add.at(vt[:, 0], idx.reshape(-1)[vis], 1)
    np.add.at(vt[:, 1], idx.reshape(-1)[~vis], 1)
    return vt


def silu(a):
    return a / (1.0 + np.exp(-a))


def expert_mlp(xe, w_gate, w_up, w_down, w4a4: bool):
    """xe [n,H] (bf16 values), w_gate/w_up [I,H], w_down [H,I] (bf16 values) -> [n,H] bf16 values."""
    if w4a4:
        xe = fake_quant(xe).astype(np.float32)
        w_gate = fake_quant(w_gate).astype(np.float32)
        w_up = fake_quant(w_up).astype(np.float32)
        w_down = fake_quant(w_down).astype(np.float32)
    g = xe @ w_gate.T
    u = xe @ w_up.T
    h = bf16_round(silu(g) * u)
    if w4a4:
        h = fake_quant(h).astype(np.float32)
    return bf16_round(h @ w_down.T)


def moe_layer(x, modality, wg, gate_up, down, k, scoring, expert_prec=None, bias=None,
              routed_scaling=1.0, norm_min=1e-12, logits=None, shared=None, partial_el=None):
    """x [T,H] bf16 values (float32); gate_up [E,2I,H] (HF: gate rows first);
    down [E,H,I]; expert_prec [E] 0/1; shared: (gate_up [2Is,H], down [H,Is]) of a
    shared-expert MLP added to every token (BF16 path, bf16 output, summed with the
    routed contributions before the one final rounding). Returns dict with y and
    intermediates."""
    T, H = x.shape
    E = wg.shape[0]
    I = down.shape[2]
    logits, idx, w = route(x, wg, k, scoring, bias, routed_scaling, norm_min, logits)
    prec = np.zeros(E, np.int64) if expert_prec is None else np.asarray(expert_prec)
    y_pairs = np.zeros((T, k, H), np.float32)
    for e in range(E):
        tok, slot = np.nonzero(idx == e)
        if len(tok) == 0:
            continue
        ye = expert_mlp(x[tok], gate_up[e, :I], gate_up[e, I:], down[e], bool(prec[e]))
        y_pairs[tok, slot] = ye
    if partial_el:
        # rank-partial return: the slots of a W4A4 owner rank d (expert e on
        # rank e // partial_el) enter as ONE bf16-rounded partial sum per (token, d)
        owner = idx // partial_el
        w4 = prec[idx].astype(bool)
        acc = (np.where(w4, 0.0, w)[:, :, None] * y_pairs).sum(axis=1, dtype=np.float32)
        for d in np.unique(owner[w4]):
            m = (w4 & (owner == d)).astype(np.float32)
            part = bf16_round(((m * w)[:, :, None] * y_pairs).sum(axis=1, dtype=np.float32))
            acc = acc + part
    else:
        acc = (w[:, :, None] * y_pairs).sum(axis=1, dtype=np.float32)
    if shared is not None:
        Is = shared[1].shape[1]
        acc = acc + expert_mlp(x, shared[0][:Is], shared[0][Is:], shared[1], False)
    out = bf16_round(acc)
    return dict(y=out, logits=logits, idx=idx, w=w, vt=expert_counts(idx, modality, E))
