"""NVFP4 block quantiser (K3/K4) — device implementation of the reference rule.

Mirrors ``moesim.fp4`` (fp4.py) on the path:
  quantize_blocks(values) -> (codes (n,16) u8, scale_bits (n,) u8)   fp4.py:173-227
  QuantizationDomainError                                              fp4.py:22
  pack_blocks / write_blocks (the 9-byte block file format)           fp4.py:246-283
and adds the product entry ``quantize_nvfp4`` which quantises a bf16 weight
matrix straight into the tcgen05 block-scaled operand layout (packed codes +
128x4-atom scale factors) on a caller-chosen stream, CTA-limited if asked.
All arithmetic runs in csrc/quant.cu; there is no host fallback.
"""

from __future__ import annotations

import struct

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


def pack_blocks(codes: np.ndarray, scale_bits: np.ndarray) -> bytes:
    """9 bytes per block: 8 code bytes (low nibble = even index) + 1 scale byte
    (pack_block, fp4.py:246-252)."""
    c = np.asarray(codes, dtype=np.uint8).reshape(-1, 16)
    s = np.asarray(scale_bits, dtype=np.uint8).reshape(-1, 1)
    packed = (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)
    return np.concatenate([packed, s], axis=1).tobytes()


def write_blocks(codes: np.ndarray, scale_bits: np.ndarray, element_count: int, path) -> None:
    """FP4REF01 file (write_blocks, fp4.py:265-270)."""
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", element_count))
        f.write(pack_blocks(codes, scale_bits))


def sf_mma_to_flat(sf_mma: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """Un-swizzle a REALB_SF_MMA128x4 scale buffer to [rows, cols/16] (host helper)."""
    nkb = cols // 16
    a = np.asarray(sf_mma, dtype=np.uint8).reshape(rows // 128, nkb // 4, 32, 4, 4)
    # a[tm, tk, r0, r1, k] with r = tm*128 + r1*32 + r0, kb = tk*4 + k
    return a.transpose(0, 3, 2, 1, 4).reshape(rows, nkb)
