"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This package is the checker for the CUDA path, never the product: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` arm may import it. The product (paper_2604_19503_b200)
never imports it and fails loudly if its CUDA extension is missing.

Contents
  fp4_oracle.c   C restatement of moesim.fp4.quantize_blocks (fp4.py:173-227),
                 built by oracle/Makefile into oracle/build/liboracle_fp4.so
  moe_ref.py     numpy restatement of the MoE-layer path (router D1 contract,
                 stats, reference policy, reference block quantiser, expert
                 MLPs in fp32, combine)
  policy_ref.py  aggregate_rank_loads + plan_realb (core.py:106-130,
                 balancers.py:89-122) in plain Python
  fp4_numpy.py   numpy float64 restatement of quantize_blocks (fp4.py:173-227),
                 the "reference quantiser" CPU baseline bench.py times
  cpu_arm.py     bench.py's CPU arms (cpu_baseline, --impl reference)

Pinning: tests/test_oracle.py checks the C oracle against fixtures generated
by running the reference itself (tests/golden/make_golden.py) and against the
reference's own golden SHA-256 (tests/test_fp4.py:194-210). The MoE-layer
parts beyond the quantiser/policy (router, GEMMs, combine) have no reference
implementation: "parity unpinned" by the reference for those,
and the oracle defines them.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle_fp4.so"
_lib = None


def build() -> Path:
    src = HERE / "fp4_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.oracle_quantize_blocks.restype = C.c_int
        L.oracle_quantize_blocks.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.oracle_dequantize_blocks.restype = None
        L.oracle_dequantize_blocks.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.oracle_quantize_bf16.restype = C.c_int
        L.oracle_quantize_bf16.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


class OracleDomainError(ValueError):
    pass


def quantize_blocks(values) -> tuple[np.ndarray, np.ndarray]:
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    if v.ndim != 2 or v.shape[1] != 16:
        raise ValueError("expected an (n, 16) array")
    n = v.shape[0]
    codes = np.zeros((n, 16), np.uint8)
    sb = np.zeros((n,), np.uint8)
    if lib().oracle_quantize_blocks(v.ctypes.data, n, codes.ctypes.data, sb.ctypes.data):
        raise OracleDomainError("block contains a non-finite value")
    return codes, sb


def dequantize_blocks(codes, scale_bits) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8).reshape(-1, 16))
    s = np.ascontiguousarray(np.asarray(scale_bits, dtype=np.uint8).reshape(-1))
    out = np.zeros(c.shape, np.float64)
    lib().oracle_dequantize_blocks(c.ctypes.data, s.ctypes.data, c.shape[0], out.ctypes.data)
    return out


def quantize_bf16(x_bits: np.ndarray):
    """bf16 bit patterns (uint16 [rows, cols]) -> packed codes [rows, cols/2], flat sf."""
    x = np.ascontiguousarray(x_bits, dtype=np.uint16)
    rows, cols = x.shape
    codes = np.zeros((rows, cols // 2), np.uint8)
    sf = np.zeros((rows, cols // 16), np.uint8)
    if lib().oracle_quantize_bf16(x.ctypes.data, rows, cols, codes.ctypes.data, sf.ctypes.data):
        raise OracleDomainError("block contains a non-finite value")
    return codes, sf


def fake_quant(x: np.ndarray) -> np.ndarray:
    """Quantise-dequantise along the last axis in 16-blocks (the reference block
    rule); x float array with last dim % 16 == 0. Returns float64."""
    shp = x.shape
    c, s = quantize_blocks(np.asarray(x, np.float64).reshape(-1, 16))
    return dequantize_blocks(c, s).reshape(shp)


def quantize_tensor(values):
    """quantize_tensor + ErrorSummary (fp4.py:137-170): flat values, the tail block
    zero-padded -> (9-byte block records uint8 [nb, 9], rmse, relative_rmse,
    per-block max relative error [nb]). The sums are sequential fp64 running sums
    in element order (np.cumsum), i.e. the reference's own accumulation order."""
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    n = v.size
    if n == 0:
        raise ValueError("values must be non-empty")
    nb = (n + 15) // 16
    pad = np.zeros(nb * 16)
    pad[:n] = v
    c, s = quantize_blocks(pad.reshape(nb, 16))
    d = dequantize_blocks(c, s).reshape(-1)[:n]
    err = v - d
    sq_err = float(np.cumsum(err * err)[-1])
    sq_val = float(np.cumsum(v * v)[-1])
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(v != 0.0, np.abs(err) / np.abs(v), 0.0)
    relp = np.zeros(nb * 16)
    relp[:n] = rel
    max_rel = relp.reshape(nb, 16).max(axis=1)
    rec = np.concatenate([(c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8), s[:, None]], axis=1)
    return rec, float(np.sqrt(sq_err / n)), (float(np.sqrt(sq_err / sq_val)) if sq_val > 0 else 0.0), max_rel
