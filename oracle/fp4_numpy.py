"""CPU ORACLE, numpy form of the reference quantiser — TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference's vectorised block quantiser
(moesim/fp4.py:173-227), step by step, with the reference's numpy primitives
(np.frexp, np.rint half-to-even, searchsorted over the E2M1 midpoints with the
odd-index tie bump). It exists for one purpose: bench.py times it on the box's
host as BASELINE.md §3's "reference quantiser" CPU baseline (the reference
itself is not present on the GPU box). Its outputs are pinned bit-exact to the
reference fixtures and to oracle/fp4_oracle.c by tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np

_MIDS = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
_SUB = 2.0 ** -9          # E4M3 minimum subnormal
_MAXF = 448.0             # E4M3 maximum finite


def _encode_scales(raw: np.ndarray, nonzero: np.ndarray) -> np.ndarray:
    """raw = amax / 6 (fp64) -> E4M3 bits (fp4.py:189-209)."""
    bits = np.zeros(raw.shape, np.uint8)
    sub = raw < 2.0 ** -6
    m_sub = np.rint(raw[sub] / _SUB).astype(np.int64)
    bits[sub] = np.minimum(m_sub, 8).astype(np.uint8)          # m == 8 rounds up to 0x08
    mant, ex = np.frexp(raw)
    e = ex.astype(np.int64) - 1
    m = np.rint((mant * 2.0 - 1.0) * 8.0).astype(np.int64)
    e = e + (m == 8)
    m[m == 8] = 0
    b = ((e + 7) << 3) | m
    b[(e > 8) | ((e == 8) & (m > 6))] = 0x7E
    norm = ~sub & (raw < _MAXF)
    bits[norm] = b[norm].astype(np.uint8)
    bits[raw >= _MAXF] = 0x7E
    bits[nonzero & (bits == 0)] = 1
    return bits


def _decode_scales(bits: np.ndarray) -> np.ndarray:
    se = (bits >> 3).astype(np.float64)
    sm = (bits & 7).astype(np.float64)
    return np.where(se == 0, sm * _SUB, (1.0 + sm / 8.0) * np.exp2(se - 7.0))


def quantize_blocks(values) -> tuple[np.ndarray, np.ndarray]:
    """(n, 16) float -> (codes uint8 (n, 16), scale bits uint8 (n,))."""
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 2 or v.shape[1] != 16:
        raise ValueError("expected an (n, 16) array")
    if not np.isfinite(v).all():
        raise ValueError("block contains a non-finite value")
    amax = np.abs(v).max(axis=1)
    nonzero = amax > 0.0
    bits = _encode_scales(amax / 6.0, nonzero)
    scale = _decode_scales(bits)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(nonzero[:, None], v / scale[:, None], 0.0)
    mag = np.abs(q)
    idx = np.searchsorted(_MIDS, mag.ravel(), side="left").reshape(mag.shape)
    at_mid = (idx < 7) & (mag == _MIDS[np.minimum(idx, 6)])
    idx = idx + (at_mid & (idx % 2 == 1))                     # ties -> even index
    codes = np.where((q < 0) & (idx > 0), idx | 8, idx).astype(np.uint8)
    return codes, bits
