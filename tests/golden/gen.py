"""Deterministic input generators shared by make_golden.py (which runs the
reference to produce expected outputs) and the parity tests (which run the
oracle / the CUDA path on the very same inputs)."""

from __future__ import annotations

import numpy as np


def fp4_regime_blocks() -> np.ndarray:
    """The six regimes of the reference test tests/test_fp4.py:124-133 (seed 42)."""
    rng = np.random.default_rng(42)
    parts = [
        rng.uniform(-1, 1, (500, 16)),
        rng.uniform(-1e-4, 1e-4, (300, 16)),  # subnormal-scale regime
        rng.uniform(-5000, 5000, (300, 16)),  # scale clamps at max finite
        rng.choice([0.0, 0.5, 1.0, 1.5, 2, 3, 4, 6, -6, -4], (300, 16)),
        np.zeros((50, 16)),
        rng.normal(0, 1, (500, 16)) * np.exp2(rng.integers(-20, 12, (500, 1)).astype(float)),
    ]
    return np.concatenate(parts)


def acceptance_blocks() -> np.ndarray:
    """tests/test_acceptance.py:353-354: 1e6 blocks U(-100, 100), seed 909."""
    return np.random.default_rng(909).uniform(-100, 100, (1_000_000, 16))


def bf16_finite_values() -> np.ndarray:
    """All finite bf16 values as float64 (65280 values; +0 and -0 both present)."""
    bits = np.arange(1 << 16, dtype=np.uint32)
    with np.errstate(invalid="ignore"):
        f = (bits << 16).view(np.float32).astype(np.float64)
    return f[np.isfinite(f)]


def bf16_amax_blocks() -> np.ndarray:
    """One block per non-negative finite bf16 amax: [amax, 0 x 15] (32641 blocks)."""
    v = bf16_finite_values()
    v = np.unique(v[v >= 0])
    out = np.zeros((len(v), 16))
    out[:, 0] = v
    return out


def bf16_code_table_blocks() -> np.ndarray:
    """Exhaustive (bf16 value x E4M3 scale) code table.

    For every scale pattern s in 1..0x7E the anchor a = 6 * decode(s) (exact in
    bf16) pins the block scale to s; every finite bf16 v with |v| <= a is then
    quantised under that scale, 15 per block after the anchor.
    """
    vals = bf16_finite_values()
    blocks = []
    for s in range(1, 0x7F):
        e, m = s >> 3, s & 7
        dec = m * 2.0**-9 if e == 0 else (1 + m / 8) * 2.0 ** (e - 7)
        a = 6.0 * dec
        sel = vals[np.abs(vals) <= a]
        pad = (-len(sel)) % 15
        sel = np.concatenate([sel, np.zeros(pad)]).reshape(-1, 15)
        blk = np.concatenate([np.full((len(sel), 1), a), sel], axis=1)
        blocks.append(blk)
    return np.concatenate(blocks)


GOLDEN_FILE_INPUT = [0.0, 0.5, -0.5, 1.0, -1.0, 1.5, -1.5, 2.0, -2.0, 3.0, -3.0, 4.0, -4.0,
                     6.0, -6.0, 0.0] + [0.25, -0.75, 1.1, 2.9] * 4
GOLDEN_FILE_SHA256 = "c49e5a408130e45b1d852bad0787ce4ac1792cc65084830a0e9be3d9975789aa"


def policy_cases(n: int = 400, seed: int = 77):
    """Random per-rank (vision, text) loads and RealbParams, with boundary cases
    (load == C * mean, v/total == M_d, sub-threshold batches, zero ranks)."""
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        R = int(rng.choice([1, 2, 4, 8]))
        kind = i % 5
        if kind == 0:
            tot = rng.integers(0, 10_000, R)
        elif kind == 1:  # exact-mean boundary: C * mean hit exactly
            tot = np.full(R, int(rng.integers(1, 500)) * R)
            tot[0] *= 2
        elif kind == 2:  # sub-threshold batches
            tot = rng.integers(0, 2048 // max(R, 1), R)
        elif kind == 3:  # zero ranks mixed in
            tot = rng.integers(0, 5_000, R) * (rng.random(R) < 0.6)
        else:  # heavy skew
            tot = (rng.pareto(1.2, R) * 1000).astype(np.int64)
        frac = rng.choice([0.0, 0.3, 0.7, 0.9, 1.0, rng.random()], R)
        v = np.rint(tot * frac).astype(np.int64)
        C = float(rng.choice([1.0, 0.5, 1.25, 2.0, 1.0 + rng.random()]))
        Md = float(rng.choice([0.0, 0.7, 0.9, 1.0, rng.random()]))
        thr = int(rng.choice([0, 2048, 2048 * 8, int(rng.integers(0, 50_000))]))
        iso = bool(rng.random() < 0.25)
        cases.append(dict(v=[int(a) for a in v], t=[int(a) for a in (tot - v)], C=C, Md=Md,
                          thr=thr, iso=iso))
    return cases


ON_GRID = GOLDEN_FILE_INPUT[:16]


def tensor_cases() -> list[np.ndarray]:
    """Flat inputs for quantize_tensor + ErrorSummary (fp4.py:137-170): the
    reference tests' cases (tests/test_fp4.py:151-179) plus ragged, wide-range and
    bf16-weight inputs."""
    rng = np.random.default_rng(2604)
    wide = rng.normal(0, 1, 1001) * np.exp2(rng.integers(-24, 14, 1001).astype(float))
    wide[rng.integers(0, 1001, 40)] = 0.0
    w = (rng.normal(0, 0.02, 4099)).astype(np.float32)
    wbf16 = ((w.view(np.uint32) + 0x7FFF + ((w.view(np.uint32) >> 16) & 1)) & 0xFFFF0000).view(np.float32)
    return [np.array(ON_GRID, float), np.full(17, 6.0), np.array([6.0] * 16 + [1.25]), np.array([1.25]),
            np.random.default_rng(0).standard_normal(4096), wide, wbf16.astype(np.float64),
            np.array(GOLDEN_FILE_INPUT, float)]
