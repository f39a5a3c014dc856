"""K4 — the activation-side NVFP4 quantiser, bit-exact with the reference block
rule (oracle.quantize_bf16: the C restatement of fp4.py:173-227) on the very
bf16 rows each producer consumed:

  realb_dispatch_permute   single-GPU layer: rows of W4A4 experts -> codes + MMA scales
  realb_ep_pack (fmt 1)    EP sender side: packed [H/2 codes][H/16 scales] rows
  realb_p2p_pack_direct    host-sync-free EP: straight into the owner's operand, scales
  + realb_sf_rows_to_mma   converted to the MMA layout there (tests/test_ep_gpu.py
                           _check_direct_dispatch_operands, every EP device-plan case)
  K6 SwiGLU epilogue       tests/test_gemm_fp4_gpu.py::test_fp4_swiglu_requant_epilogue

The token rows span the quantiser's regimes (subnormal and saturating scales,
an all-zero row, exact E2M1 ties) so every branch of the rule is exercised.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
from paper_2604_19503_b200.quant import sf_mma_to_flat
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

pytestmark = pytest.mark.gpu


def _regime_rows(x: torch.Tensor, seed: int) -> torch.Tensor:
    """Scale token rows into the reference quantiser's regimes: tiny (subnormal
    E4M3 scales), huge (saturating at 448), an all-zero row, and a row of exact
    E2M1 midpoints x 2^k (ties)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    T, H = x.shape
    f = torch.tensor([1e-6, 3e-4, 1.0, 1.0, 7.0, 4000.0, 5e4])[torch.randint(0, 7, (T,), generator=g)]
    y = (x.float().cpu() * f[:, None]).to(torch.bfloat16)
    y[0] = 0
    if T > 1:
        mids = torch.tensor([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, -0.75])
        y[1] = (mids.repeat(H // 8) * 2.0 ** -3).to(torch.bfloat16)
    return y.to(x.device)


def _layer(name, E, T, seed=2024):
    from dataclasses import replace

    shape = replace(SHAPES[name], num_experts=E or SHAPES[name].num_experts)
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=1, seed=seed))
    gu, dn = make_experts(shape, seed=seed)
    bias = torch.zeros(shape.num_experts, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
    layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn, bias=bias), max_tokens=T)
    return shape, layer, _regime_rows(x, seed), mod


def _oracle_rows(x: torch.Tensor):
    return oracle.quantize_bf16(x.view(torch.int16).cpu().numpy().view(np.uint16))


@pytest.mark.parametrize("name,E,T", [("tiny", None, 1024), ("kimi", 16, 700), ("qwen", 32, 333)])
def test_dispatch_permute_w4a4_rows_bit_exact(name, E, T):
    shape, layer, x, mod = _layer(name, E, T)
    E, k, H = shape.num_experts, shape.top_k, shape.hidden
    layer.route(x, mod)
    prec = np.zeros(E, np.uint8)
    prec[::2] = _lib.PREC_W4A4  # mixed: every other expert W4A4
    layer.prec_dev.copy_(torch.from_numpy(prec))
    layer.align(T)
    ws = layer._fp4_ws()
    _lib.call("realb_dispatch_permute", x.data_ptr(), layer.topk_idx.data_ptr(), T, H, E, k,
              layer.prec_dev.data_ptr(), layer.layout.data_ptr(), (T + 63) // 64, layer.rows_cap,
              layer.pair_pos.data_ptr(), layer.a_bf16.data_ptr(), ws["a_codes"].data_ptr(),
              ws["a_sf"].data_ptr(), layer.flag.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    layer.check_flag()
    idx = layer.topk_idx[:T].cpu().numpy()
    pos = layer.pair_pos[:T].cpu().numpy()
    codes = ws["a_codes"].cpu().numpy()
    sf = sf_mma_to_flat(ws["a_sf"].cpu().numpy(), layer.rows_cap, H)
    oc, osf = _oracle_rows(x)
    t, j = np.nonzero(prec[idx] == _lib.PREC_W4A4)
    assert len(t) > 0
    p = pos[t, j]
    assert (codes[p] == oc[t]).all()
    assert (sf[p] == osf[t]).all()
    # the W16A16 experts' rows are the bf16 tokens, untouched
    t16, j16 = np.nonzero(prec[idx] != _lib.PREC_W4A4)
    a = layer.a_bf16.view(torch.int16).cpu().numpy()
    assert (a[pos[t16, j16]] == x.view(torch.int16).cpu().numpy()[t16]).all()


@pytest.mark.parametrize("name,E,T,R", [("tiny", None, 1024, 2), ("kimi", 16, 700, 4), ("qwen", 32, 333, 8)])
def test_ep_pack_nvfp4_rows_bit_exact(name, E, T, R):
    """realb_ep_pack with mixed destination formats: fmt-1 rows are the oracle's
    codes followed by its scales; fmt-0 rows are the bf16 token."""
    shape, layer, x, mod = _layer(name, E, T)
    E, k, H = shape.num_experts, shape.top_k, shape.hidden
    El = E // R
    layer.route(x, mod)
    layer.prec_dev.zero_()
    layer.align(T, row_align=1)
    torch.cuda.synchronize()
    idx = layer.topk_idx[:T].cpu().numpy()
    counts = np.bincount(idx.reshape(-1) // El, minlength=R).astype(np.int64)
    fmt = np.array([(d + 1) % 2 for d in range(R)], np.uint8)  # ranks 0, 2, ... NVFP4
    units = np.array([H // 2 + H // 16 if f else 2 * H for f in fmt], np.int64)
    row0 = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    byte0 = np.concatenate([[0], np.cumsum(counts * units)[:-1]]).astype(np.int64)
    send = torch.zeros(int((counts * units).sum()) + 16, dtype=torch.uint8, device="cuda")
    pos_t = torch.empty(T, k, dtype=torch.int32, device="cuda")
    _lib.call("realb_ep_pack", x.data_ptr(), layer.topk_idx.data_ptr(), T, H, E, k, layer.layout.data_ptr(),
              (T + 63) // 64, R, fmt.ctypes.data, row0.ctypes.data, byte0.ctypes.data, pos_t.data_ptr(),
              send.data_ptr(), layer.flag.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    layer.check_flag()
    buf = send.cpu().numpy()
    pos = pos_t.cpu().numpy()
    oc, osf = _oracle_rows(x)
    xb = x.view(torch.int16).cpu().numpy().view(np.uint8).reshape(T, 2 * H)
    n4 = n16 = 0
    for t in range(T):
        for j in range(k):
            d = int(idx[t, j]) // El
            off = int(byte0[d] + (int(pos[t, j]) - int(row0[d])) * units[d])
            row = buf[off:off + units[d]]
            if fmt[d]:
                assert (row[:H // 2] == oc[t]).all(), (t, j)
                assert (row[H // 2:] == osf[t]).all(), (t, j)
                n4 += 1
            else:
                assert (row == xb[t]).all(), (t, j)
                n16 += 1
    assert n4 > 0 and n16 > 0
