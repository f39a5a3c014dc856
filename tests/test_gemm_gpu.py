"""K5: grouped BF16 tcgen05 GEMM vs a plain PyTorch fp32 reference."""

import numpy as np
import pytest
import torch

from helpers import host_layout
from paper_2604_19503_b200 import _lib

pytestmark = pytest.mark.gpu


def run_bf16(A, W, lay, N, K, E, prec, epi, rows_cap):
    dev = A.device
    lay_t = torch.from_numpy(lay).to(dev)
    NO = N if epi == _lib.EPI_STORE else N // 2
    out = torch.full((rows_cap, NO), float("nan"), dtype=torch.bfloat16, device=dev)
    _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows_cap, N, K, E,
              lay_t.data_ptr(), prec, epi, out.data_ptr(), 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    return out


def ref_rows(A, W, lay, E, N, counts, prec_sel, prec, epi):
    outs = {}
    for e in range(E):
        if prec_sel[e] != prec or counts[e] == 0:
            continue
        rs = int(lay[8 + e])
        a = A[rs:rs + counts[e]].float()
        y = a @ W[e * N:(e + 1) * N].float().T
        if epi == _lib.EPI_SWIGLU:
            nb = N // 256
            y = y.view(-1, nb, 2, 128)
            g, u = y[:, :, 0], y[:, :, 1]
            y = (torch.nn.functional.silu(g) * u).reshape(-1, N // 2)
        outs[e] = (rs, y)
    return outs


@pytest.fixture(params=["1", "2"], ids=["cta1", "pair"])
def cluster(request, monkeypatch):
    """Both kernel forms: one CTA per tile, and 2-CTA pairs (cta_group::2, M = 256)."""
    monkeypatch.setenv("REALB_GEMM_CLUSTER", request.param)
    return request.param


@pytest.mark.parametrize("E,N,K,counts", [
    (1, 256, 64, [128]),
    (1, 256, 128, [77]),
    (4, 512, 2048, [300, 0, 17, 1000]),
    (8, 2816, 2048, [513, 129, 1, 0, 777, 256, 2048, 90]),   # Kimi gate_up shape
    (8, 2048, 1408, [513, 129, 1, 0, 777, 256, 2048, 90]),   # Kimi down shape
])
@pytest.mark.parametrize("epi", [_lib.EPI_STORE, _lib.EPI_SWIGLU])
def test_grouped_bf16(E, N, K, counts, epi, cluster, parity_log):
    torch.manual_seed(E * 31 + N + K)
    prec_sel = np.zeros(E, np.int64)
    lay, rows = host_layout(counts, prec_sel)
    rows_cap = max(rows, 128)
    A = torch.randn(rows_cap, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
    out = run_bf16(A, W, lay, N, K, E, 0, epi, rows_cap)
    for e, (rs, y) in ref_rows(A, W, lay, E, N, counts, prec_sel, 0, epi).items():
        got = out[rs:rs + counts[e]].float()
        # against the fp32 reference rounded to bf16 (the kernel's one output rounding):
        # what remains is fp32 accumulation order (+ __expf in SwiGLU) flipping roundings
        yb = y.to(torch.bfloat16).float()
        err = float((got - yb).norm() / yb.norm().clamp_min(1e-30))
        parity_log("k5_vs_fp32_torch_bf16_rounded", err, 2e-3)
        assert err < 2e-3, (e, err)


def test_grouped_bf16_precision_subset():
    """Only groups of the requested precision class are computed."""
    E, N, K = 4, 256, 256
    counts = [200, 300, 100, 50]
    prec_sel = np.array([0, 1, 0, 1])
    lay, rows = host_layout(counts, prec_sel)
    A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") / 16).to(torch.bfloat16)
    out = run_bf16(A, W, lay, N, K, E, 1, _lib.EPI_STORE, rows)
    for e in range(E):
        rs = int(lay[8 + e])
        blk = out[rs:rs + counts[e]]
        if prec_sel[e] == 1:
            y = A[rs:rs + counts[e]].float() @ W[e * N:(e + 1) * N].float().T
            assert ((blk.float() - y).norm() / y.norm()) < 1e-2
        else:
            assert torch.isnan(blk.float()).all()


@pytest.mark.parametrize("E,N,K,counts,T", [
    (1, 256, 64, [77], 50),
    (4, 512, 2048, [300, 0, 17, 1000], 700),
    (8, 2816, 2048, [513, 129, 1, 0, 777, 256, 2048, 90], 1500),   # Kimi gate_up shape
    (8, 2048, 1408, [513, 129, 1, 0, 777, 256, 2048, 90], 3000),   # Kimi down shape
])
@pytest.mark.parametrize("epi", [_lib.EPI_STORE, _lib.EPI_SWIGLU])
def test_grouped_bf16_gather_equals_copy(E, N, K, counts, T, epi):
    """The gather form (A rows read from x through row_src by TMA tile::gather4)
    gives bit-for-bit the rows the grouped-operand form gives on the copied rows
    (same MMAs in the same order); padding rows repeat valid rows of their tile
    (activation-like operands), so their outputs are finite."""
    torch.manual_seed(E + N + K + T)
    prec_sel = np.zeros(E, np.int64)
    lay, rows = host_layout(counts, prec_sel)
    rows_cap = max(rows, 128)
    x = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    src = torch.randint(0, T, (rows_cap,), dtype=torch.int32, device="cuda")
    W = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
    A = x[src.long()].contiguous()
    ref = run_bf16(A, W, lay, N, K, E, 0, epi, rows_cap)
    lay_t = torch.from_numpy(lay).cuda()
    NO = N if epi == _lib.EPI_STORE else N // 2
    out = torch.full((rows_cap, NO), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.call("realb_grouped_gemm_bf16_gather", x.data_ptr(), T, src.data_ptr(), W.data_ptr(), rows_cap, N, K,
              E, lay_t.data_ptr(), 0, epi, out.data_ptr(), 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    for e in range(E):
        rs = int(lay[8 + e])
        c = counts[e]
        assert torch.equal(out[rs:rs + c], ref[rs:rs + c]), e
        pad = (c + 127) // 128 * 128
        if pad > c:  # padding rows repeat valid rows of their tile: finite, never NaN garbage
            assert torch.isfinite(out[rs + c:rs + pad].float()).all(), e


@pytest.mark.parametrize("E,N,K,counts,n_dst", [
    (4, 512, 2048, [300, 0, 17, 1000], 3),
    (8, 2048, 1408, [513, 129, 1, 0, 777, 256, 2048, 90], 8),   # Kimi down shape, EP8
])
def test_grouped_bf16_scatter_equals_store(E, N, K, counts, n_dst):
    """realb_grouped_gemm_bf16_scatter (the down GEMM fused with the EP return):
    every valid row lands bit-identical to the STORE epilogue's row at its mapped
    (destination, row); rows of other destinations / padding are not written."""
    torch.manual_seed(E + N)
    prec_sel = np.zeros(E, np.int64)
    lay, rows = host_layout(counts, prec_sel)
    rows_cap = max(rows, 128)
    A = torch.randn(rows_cap, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
    ref = run_bf16(A, W, lay, N, K, E, 0, _lib.EPI_STORE, rows_cap).cpu()
    rng = np.random.default_rng(E)
    valid = np.concatenate([int(lay[8 + e]) + np.arange(c) for e, c in enumerate(counts)])
    d = rng.integers(0, n_dst, len(valid))
    m = np.full(rows_cap, -1, np.int32)
    sizes = []
    for dd in range(n_dst):
        sel = valid[d == dd]
        m[sel] = (dd << 25) | rng.permutation(len(sel))
        sizes.append(len(sel))
    dsts = [torch.full((s + 1, N), 7.0, dtype=torch.bfloat16, device="cuda") for s in sizes]
    bases = np.array([t.data_ptr() for t in dsts], np.uint64)
    lay_t = torch.from_numpy(lay).cuda()
    m_t = torch.from_numpy(m).cuda()
    _lib.call("realb_grouped_gemm_bf16_scatter", A.data_ptr(), W.data_ptr(), rows_cap, N, K, E, lay_t.data_ptr(),
              0, m_t.data_ptr(), n_dst, bases.ctypes.data, 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    got = [t.cpu() for t in dsts]
    for g in valid:
        dd, j = int(m[g]) >> 25, int(m[g]) & ((1 << 25) - 1)
        assert torch.equal(got[dd][j], ref[g]), (g, dd, j)
    for dd, s in enumerate(sizes):
        assert (got[dd][s:].float() == 7.0).all()
