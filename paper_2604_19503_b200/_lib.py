"""ctypes binding of the C-ABI library ``lib/librealb_b200.so`` (include/realb.h).

The library is the product path: there is no CPU or PyTorch fallback. Loading
fails loudly (``RealbUnavailable``) if the library was not built, and every
call maps a negative status to ``RealbError`` carrying ``realb_last_error()``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "librealb_b200.so"

OK = 0
EINVAL = -1
ECUDA = -2
EUNSUPPORTED = -3

DT_BF16, DT_F32, DT_F64 = 0, 1, 2
SF_FLAT, SF_MMA128x4 = 0, 1
SCORE_SOFTMAX_RENORM, SCORE_SIGMOID_RENORM, SCORE_SOFTMAX_CLAMPNORM = 0, 1, 2
PREC_W16A16, PREC_W4A4 = 0, 1
EPI_STORE, EPI_SWIGLU = 0, 1


class RealbUnavailable(RuntimeError):
    """The sm_100a extension is missing; there is deliberately no fallback."""


class RealbError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


_vp, _i32, _i64, _f32, _f64, _u32 = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double, C.c_uint32

# name -> (restype, argtypes); must list every function of include/realb.h
SIGNATURES: dict[str, tuple] = {
    "realb_abi_version": (_i32, []),
    "realb_last_error": (C.c_char_p, []),
    "realb_num_sms": (_i32, []),
    "realb_quantize_nvfp4": (_i32, [_vp, _i32, _i64, _i64, _vp, _vp, _i32, _vp, _i32, _vp]),
    "realb_router_topk_stats": (
        _i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _f32, _f32, _vp, _vp, _vp, _vp, _vp]),
    "realb_layout_words": (_i64, [_i32, _i32]),
    "realb_moe_align_plan": (_i32, [_vp, _i32, _i32, _i32, _i32, _f64, _f64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "realb_quantize_experts_nvfp4": (_i32, [_vp, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp]),
    "realb_quantize_experts2_nvfp4": (
        _i32, [_vp, _i64, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _i32, _vp]),
    "realb_quantize_tensor_nvfp4": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp]),
    "realb_dequantize_blocks": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "realb_moe_align": (_i32, [_vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp]),
    "realb_gather_rows": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "realb_ep_regroup": (_i32, [_vp, _i32, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "realb_index_rows": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "realb_dispatch_permute": (
        _i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "realb_grouped_gemm_bf16": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _i32, _vp]),
    "realb_grouped_gemm_bf16_gather": (
        _i32, [_vp, _i64, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _i32, _vp]),
    "realb_grouped_gemm_bf16_copyin": (
        _i32, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "realb_grouped_gemm_bf16_scatter": (
        _i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _i32, _vp]),
    "realb_grouped_gemm_nvfp4_scatter": (
        _i32, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _i32, _vp, _i32, _vp]),
    "realb_p2p_return_map": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "realb_sf_rows_to_mma": (_i32, [_vp, _i64, _i32, _vp, _i32, _i32, _vp, _vp]),
    "realb_dispatch_index": (
        _i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "realb_grouped_gemm_nvfp4": (
        _i32, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _vp, _i32, _vp]),
    "realb_combine": (_i32, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "realb_combine_partial": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _i64, _i64, _vp, _vp]),
    "realb_plan": (_i32, [_vp, _i32, _f64, _f64, _i64, _i32, _vp, _vp]),
    "realb_ep_pack": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp,
                             _vp]),
    "realb_gather_rows_nvfp4_packed": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "realb_p2p_plan_bytes": (_i64, []),
    "realb_p2p_plan_layout": (_i32, [_vp]),
    "realb_p2p_wait_next": (_i32, [_vp, _u32, _vp, _vp, _vp]),
    "realb_p2p_publish": (_i32, [_vp, _i32, _i32, _vp, _i64, _vp]),
    "realb_p2p_plan_offsets": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "realb_p2p_pack_dev": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "realb_p2p_return_dev": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "realb_p2p_pack_direct": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp]),
    "realb_p2p_pack_direct_partial": (_i32, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp,
                                             _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp]),
    "realb_p2p_partial_return": (_i32, [_vp, _vp, _vp, _i32, _i64, _i32, _i32, _i32, _vp, _i64, _vp, _vp]),
    "realb_ipc_alloc": (_i32, [_i64, _vp, _vp]),
    "realb_ipc_open": (_i32, [_vp, _vp]),
    "realb_ipc_close": (_i32, [_vp]),
    "realb_ipc_free": (_i32, [_vp]),
    "realb_p2p_pack": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                              _vp]),
    "realb_p2p_return": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "realb_p2p_signal": (_i32, [_vp, _i32, _vp]),
    "realb_p2p_wait": (_i32, [_vp, _u32, _vp, _vp]),
}

_lib: C.CDLL | None = None

# kernels launched per successful call (realb_dispatch_permute: positions + rows)
LAUNCHES_KERNEL = {
    "realb_dispatch_permute": 2,
    "realb_quantize_nvfp4": 1, "realb_router_topk_stats": 1, "realb_moe_align": 1,
    "realb_moe_align_plan": 1, "realb_quantize_experts_nvfp4": 1, "realb_quantize_experts2_nvfp4": 1,
    "realb_grouped_gemm_bf16": 1, "realb_grouped_gemm_bf16_gather": 1, "realb_grouped_gemm_nvfp4": 1,
    "realb_grouped_gemm_bf16_copyin": 1, "realb_grouped_gemm_bf16_scatter": 1, "realb_grouped_gemm_nvfp4_scatter": 1, "realb_p2p_return_map": 1, "realb_sf_rows_to_mma": 1,
    "realb_dispatch_index": 1,  # + 1 when NVFP4 rows are quantised (call() adds it)
    "realb_combine": 1, "realb_combine_partial": 1, "realb_quantize_tensor_nvfp4": 1, "realb_dequantize_blocks": 1,
    "realb_gather_rows": 1, "realb_ep_regroup": 2, "realb_index_rows": 1,
    "realb_ep_pack": 2, "realb_gather_rows_nvfp4_packed": 1,
    "realb_p2p_pack": 2, "realb_p2p_return": 1, "realb_p2p_signal": 1, "realb_p2p_wait": 1,
    "realb_p2p_publish": 1, "realb_p2p_plan_offsets": 1, "realb_p2p_pack_dev": 2, "realb_p2p_return_dev": 1,
    "realb_p2p_wait_next": 1, "realb_p2p_pack_direct": 2, "realb_p2p_pack_direct_partial": 2,
    "realb_p2p_partial_return": 1,
}
launch_count = 0  # kernels launched through this binding (bench.py's gpu_launches)


def load() -> C.CDLL:
    """Load (once) and type the library. Raises RealbUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("REALB_LIB", LIB_PATH))
    if not path.exists():
        raise RealbUnavailable(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.realb_abi_version() != 1:
        raise RealbUnavailable("ABI version mismatch")
    _lib = lib
    return lib


def call(name: str, *args) -> int:
    global launch_count
    lib = load()
    st = getattr(lib, name)(*args)
    if st < 0:
        raise RealbError(name, st, lib.realb_last_error().decode(errors="replace"))
    launch_count += LAUNCHES_KERNEL.get(name, 0)
    if name == "realb_dispatch_index" and args[12] is not None and args[2] > 0:
        launch_count += 1
    return st


def ptr(t) -> int | None:
    """Raw data pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
