"""NVFP4 block quantiser (K3/K4) — device implementation of the reference rule.

Mirrors ``moesim.fp4`` (fp4.py) on the path:
  quantize_blocks(values) -> (codes (n,16) u8, scale_bits (n,) u8)   fp4.py:173-227
  dequantize_blocks(codes, scale_bits) -> (n,16) float64               fp4.py:230-243
  Fp4Block, quantize_block, dequantize_block                          fp4.py:90-127
  ErrorSummary, quantize_tensor                                       fp4.py:130-170
  QuantizationDomainError                                              fp4.py:22
  pack_block / unpack_block / write_blocks / read_blocks (FP4REF01)   fp4.py:246-283
and adds the product entry ``quantize_nvfp4`` which quantises a bf16 weight
matrix straight into the tcgen05 block-scaled operand layout (packed codes +
128x4-atom scale factors) on a caller-chosen stream, CTA-limited if asked.
All arithmetic runs in csrc/quant.cu; there is no host fallback.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib

BLOCK_SIZE = 16
MAGIC = b"FP4REF01"


class QuantizationDomainError(ValueError):
    """Non-finite input to the quantiser (fp4.py:22)."""


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise _lib.RealbUnavailable("the NVFP4 quantiser runs on a CUDA device; none is visible")
    return torch


_DT = {"torch.bfloat16": _lib.DT_BF16, "torch.float32": _lib.DT_F32, "torch.float64": _lib.DT_F64}


def quantize_nvfp4(x, *, layout: str = "mma", codes=None, sf=None, flag=None, max_ctas: int = 0,
                   stream=None, check: bool = True):
    """Quantise a 2-D CUDA tensor (bf16/f32/f64, cols % 16 == 0) block-wise along rows.

    Returns ``(codes, sf)``: codes uint8 [rows, cols/2] (element 2i in the low nibble),
    sf uint8 E4M3 scales, [rows, cols/16] for layout="flat" or the tcgen05 128x4-atom
    layout for layout="mma". With ``check`` the non-finite flag is read back (one sync)
    and ``QuantizationDomainError`` raised; pass ``check=False`` plus your own ``flag``
    tensor to keep the call asynchronous.
    """
    torch = _torch()
    if x.dim() != 2 or not x.is_cuda:
        raise ValueError("expected a 2-D CUDA tensor")
    dt = _DT.get(str(x.dtype))
    if dt is None:
        raise ValueError(f"unsupported dtype {x.dtype}")
    x = x.contiguous()
    rows, cols = x.shape
    if cols % BLOCK_SIZE:
        raise ValueError(f"cols must be a multiple of {BLOCK_SIZE}")
    lay = _lib.SF_MMA128x4 if layout == "mma" else _lib.SF_FLAT
    if codes is None:
        codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device=x.device)
    if sf is None:
        sf = torch.empty((rows * cols // 16,), dtype=torch.uint8, device=x.device)
        if lay == _lib.SF_FLAT:
            sf = sf.view(rows, cols // 16)
    own_flag = flag is None
    if own_flag:
        flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.call("realb_quantize_nvfp4", _lib.ptr(x), dt, rows, cols, _lib.ptr(codes), _lib.ptr(sf),
              lay, _lib.ptr(flag), int(max_ctas), _lib.stream_ptr(stream))
    if check and int(flag.item()) != 0:
        raise QuantizationDomainError("block contains a non-finite value")
    return codes, sf


def unpack_codes(packed: np.ndarray) -> np.ndarray:
    """[.., m] packed bytes -> [.., 2m] codes (low nibble first)."""
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.shape[:-1] + (p.shape[-1] * 2,), dtype=np.uint8)
    out[..., 0::2] = p & 0xF
    out[..., 1::2] = p >> 4
    return out


def quantize_blocks(values) -> tuple[np.ndarray, np.ndarray]:
    """Batch quantiser on the GPU, bit-exact with moesim.fp4.quantize_blocks.

    ``values``: (n, 16) array-like (float64 semantics are preserved: the device
    path computes in fp64 for float64 input). Returns numpy (codes (n,16), scale_bits (n,)).
    """
    torch = _torch()
    if isinstance(values, torch.Tensor):
        t = values
    else:
        arr = np.asarray(values, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[1] != BLOCK_SIZE:
            raise ValueError(f"expected an (n, {BLOCK_SIZE}) array")
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dim() != 2 or t.shape[1] != BLOCK_SIZE:
        raise ValueError(f"expected an (n, {BLOCK_SIZE}) array")
    n = t.shape[0]
    if n == 0:
        return np.zeros((0, 16), np.uint8), np.zeros((0,), np.uint8)
    t = t.to("cuda")
    codes, sf = quantize_nvfp4(t, layout="flat")
    return unpack_codes(codes.cpu().numpy()), sf.cpu().numpy().reshape(n)


@dataclass(frozen=True)
class Fp4Block:
    """One quantised block: 16 four-bit codes + an E4M3 scale pattern (fp4.py:90-105)."""

    codes: tuple[int, ...]
    scale_bits: int

    def __post_init__(self):
        if len(self.codes) != BLOCK_SIZE:
            raise ValueError(f"block must hold exactly {BLOCK_SIZE} codes")
        if any(not 0 <= c <= 0xF for c in self.codes):
            raise ValueError("codes must be 4-bit values")
        if not 0 <= self.scale_bits <= 0x7F:
            raise ValueError("scale must be a non-negative E4M3 pattern")

    @property
    def scale(self) -> float:
        return float(dequantize_blocks(np.full((1, 16), 2, np.uint8), np.array([self.scale_bits], np.uint8))[0, 0])


@dataclass(frozen=True)
class ErrorSummary:
    """quantize_tensor's error statistics over the unpadded elements (fp4.py:130-135)."""

    rmse: float
    relative_rmse: float
    max_relative_error_per_block: tuple[float, ...]


def dequantize_blocks(codes, scale_bits) -> np.ndarray:
    """(n,16) codes + (n,) scale bits -> (n,16) float64, code magnitude x scale,
    decoded on the device (realb_dequantize_blocks)."""
    torch = _torch()
    c = np.asarray(codes, dtype=np.uint8).reshape(-1, BLOCK_SIZE)
    sb = np.ascontiguousarray(np.asarray(scale_bits, dtype=np.uint8).reshape(-1))
    n = c.shape[0]
    if sb.shape[0] != n:
        raise ValueError("one scale per block expected")
    if n == 0:
        return np.zeros((0, BLOCK_SIZE), np.float64)
    packed = np.ascontiguousarray((c[:, 0::2] & 0xF) | ((c[:, 1::2] & 0xF) << 4)).astype(np.uint8)
    dc = torch.from_numpy(packed).cuda()
    ds = torch.from_numpy(sb).cuda()
    out = torch.empty(n, BLOCK_SIZE, dtype=torch.float64, device="cuda")
    _lib.call("realb_dequantize_blocks", dc.data_ptr(), ds.data_ptr(), n, _lib.DT_F64, out.data_ptr(),
              _lib.stream_ptr())
    return out.cpu().numpy()


def quantize_block(values) -> Fp4Block:
    """One block of 16 values (fp4.py:108-122)."""
    values = list(values)
    if len(values) != BLOCK_SIZE:
        raise ValueError(f"block must hold exactly {BLOCK_SIZE} values")
    c, sb = quantize_blocks(np.array([values], np.float64))
    return Fp4Block(tuple(int(v) for v in c[0]), int(sb[0]))


def dequantize_block(block: Fp4Block) -> list[float]:
    return dequantize_blocks(np.array([block.codes], np.uint8), np.array([block.scale_bits], np.uint8))[0].tolist()


def quantize_tensor_device(x, sums=None, with_blocks: bool = True):
    """Device form of quantize_tensor (realb_quantize_tensor_nvfp4) on a flat CUDA
    tensor (bf16 / f32 / f64, any length > 0): -> (records uint8 [nb, 9] (the
    FP4REF01 block records), per-block max relative error fp64 [nb] or None,
    sums fp64 [2] = (sum (x-d)^2, sum x^2)). Stream-ordered, no sync; the
    non-finite check is left to the caller (``flag`` in the returned dict)."""
    torch = _torch()
    x = x.reshape(-1)
    if not x.is_cuda:
        raise ValueError("expected a CUDA tensor")
    dt = _DT.get(str(x.dtype))
    if dt is None:
        raise ValueError(f"unsupported dtype {x.dtype}")
    n = x.numel()
    if n == 0:
        raise ValueError("values must be non-empty")
    x = x.contiguous()
    nb = (n + BLOCK_SIZE - 1) // BLOCK_SIZE
    rec = torch.empty(nb, 9, dtype=torch.uint8, device=x.device)
    mr = torch.empty(nb, dtype=torch.float64, device=x.device) if with_blocks else None
    if sums is None:
        sums = torch.zeros(2, dtype=torch.float64, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.call("realb_quantize_tensor_nvfp4", x.data_ptr(), dt, n, rec.data_ptr(), _lib.ptr(mr), sums.data_ptr(),
              flag.data_ptr(), _lib.stream_ptr())
    return {"records": rec, "max_rel": mr, "sums": sums, "flag": flag, "n": n}


def weight_error_summary(tensors) -> dict:
    """The FP4 weight-error proxy of a W4A4 rank: quantize_tensor's statistics
    (fp4.py:137-170) over a list of CUDA weight tensors (blocks of 16 along each
    row, the same blocks K3 quantises), reduced on the device. -> rmse,
    relative_rmse, and the max / mean over blocks of the per-block max relative
    error; raises QuantizationDomainError on non-finite weights."""
    torch = _torch()
    sums = None
    n, nb = 0, 0
    maxes, totals, flags = [], [], []
    for t in tensors:
        r = quantize_tensor_device(t, sums=sums)
        sums = r["sums"]
        n += r["n"]
        nb += r["max_rel"].numel()
        maxes.append(r["max_rel"].max())
        totals.append(r["max_rel"].sum())
        flags.append(r["flag"])
    if n == 0:
        return {"elements": 0}
    if int(torch.cat(flags).sum().item()) != 0:
        raise QuantizationDomainError("block contains a non-finite value")
    s = summary_from_sums(sums, n)
    return {"elements": n, "blocks": nb, "rmse": s.rmse, "relative_rmse": s.relative_rmse,
            "max_block_max_relative_error": float(torch.stack(maxes).max()),
            "mean_block_max_relative_error": float(torch.stack(totals).sum()) / nb}


def summary_from_sums(sums, n: int, max_rel=()) -> ErrorSummary:
    s = [float(v) for v in (sums.tolist() if hasattr(sums, "tolist") else sums)]
    return ErrorSummary(math.sqrt(s[0] / n), math.sqrt(s[0] / s[1]) if s[1] > 0 else 0.0, tuple(max_rel))


def quantize_tensor(values, block_size: int = BLOCK_SIZE) -> tuple[list[Fp4Block], ErrorSummary]:
    """Blockwise quantisation of a flat sequence, the last block zero-padded, with
    the error statistics over the unpadded elements (fp4.py:137-170); computed on
    the device in fp64 (the reference's arithmetic)."""
    torch = _torch()
    if block_size != BLOCK_SIZE:
        raise ValueError("only block size 16 is supported")
    if isinstance(values, torch.Tensor):
        t = values.reshape(-1)
    else:
        arr = np.asarray(list(values), dtype=np.float64)
        if arr.size == 0:
            raise ValueError("values must be non-empty")
        t = torch.from_numpy(arr)
    if t.numel() == 0:
        raise ValueError("values must be non-empty")
    r = quantize_tensor_device(t.cuda())
    if int(r["flag"].item()) != 0:
        raise QuantizationDomainError("block contains a non-finite value")
    rec = r["records"].cpu().numpy()
    blocks = [unpack_block(bytes(row)) for row in rec]
    return blocks, summary_from_sums(r["sums"], r["n"], r["max_rel"].cpu().numpy().tolist())


def pack_block(block: Fp4Block) -> bytes:
    """8 code bytes (two codes per byte, low nibble = even index) + 1 scale byte."""
    return pack_blocks(np.array([block.codes], np.uint8), np.array([block.scale_bits], np.uint8))


def unpack_block(data: bytes) -> Fp4Block:
    """9-byte record -> Fp4Block (fp4.py:255-262)."""
    if len(data) != 9:
        raise ValueError("packed block must be 9 bytes")
    b = np.frombuffer(bytes(data[:8]), np.uint8)
    codes = np.empty(16, np.uint8)
    codes[0::2], codes[1::2] = b & 0xF, b >> 4
    return Fp4Block(tuple(int(c) for c in codes), int(data[8]))


def read_blocks(path) -> tuple[list[Fp4Block], int]:
    """FP4REF01 file -> (blocks, element count) (fp4.py:273-283)."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != MAGIC:
        raise ValueError("bad magic in FP4 block file")
    (count,) = struct.unpack("<Q", data[8:16])
    body = data[16:]
    if len(body) % 9 != 0:
        raise ValueError("truncated FP4 block file")
    return [unpack_block(body[i:i + 9]) for i in range(0, len(body), 9)], count


def pack_blocks(codes: np.ndarray, scale_bits: np.ndarray) -> bytes:
    """9 bytes per block: 8 code bytes (low nibble = even index) + 1 scale byte
    (pack_block, fp4.py:246-252)."""
    c = np.asarray(codes, dtype=np.uint8).reshape(-1, 16)
    s = np.asarray(scale_bits, dtype=np.uint8).reshape(-1, 1)
    packed = (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)
    return np.concatenate([packed, s], axis=1).tobytes()


def write_blocks(*args) -> None:
    """FP4REF01 file (write_blocks, fp4.py:265-270). Two call forms:
    write_blocks(blocks: list[Fp4Block], element_count, path)        (the reference's)
    write_blocks(codes (n,16), scale_bits (n,), element_count, path) (array form)."""
    if len(args) == 3:
        blocks, element_count, path = args
        body = b"".join(pack_block(b) for b in blocks)
    elif len(args) == 4:
        codes, scale_bits, element_count, path = args
        body = pack_blocks(codes, scale_bits)
    else:
        raise TypeError("write_blocks(blocks, element_count, path) or write_blocks(codes, scale_bits, count, path)")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", element_count))
        f.write(body)


def sf_mma_to_flat(sf_mma: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """Un-swizzle a REALB_SF_MMA128x4 scale buffer to [rows, cols/16] (host helper)."""
    nkb = cols // 16
    a = np.asarray(sf_mma, dtype=np.uint8).reshape(rows // 128, nkb // 4, 32, 4, 4)
    # a[tm, tk, r0, r1, k] with r = tm*128 + r1*32 + r0, kb = tk*4 + k
    return a.transpose(0, 3, 2, 1, 4).reshape(rows, nkb)
