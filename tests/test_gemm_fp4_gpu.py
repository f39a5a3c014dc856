"""K6: grouped NVFP4 tcgen05 GEMM vs fp32 matmul of the reference-rule
dequantised operands (the FP4-emulating oracle), and the fused SwiGLU + NVFP4
re-quantisation epilogue vs the oracle block rule."""

import numpy as np
import pytest
import torch

import oracle
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from oracle.moe_ref import bf16_round
from paper_2604_19503_b200.quant import quantize_nvfp4, sf_mma_to_flat, unpack_codes

pytestmark = pytest.mark.gpu

MAGS = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6, -0.0, -0.5, -1, -1.5, -2, -3, -4, -6], np.float64)


def decode_e4m3(b):
    b = np.asarray(b, np.int64)
    e, m = b >> 3, b & 7
    return np.where(e == 0, m * 2.0**-9, (1 + m / 8) * 2.0 ** (e - 7))


def dequant(codes_packed, sf_mma, rows, cols):
    c = unpack_codes(codes_packed.cpu().numpy()).reshape(rows, cols)
    s = sf_mma_to_flat(sf_mma.cpu().numpy(), rows, cols)
    return MAGS[c] * np.repeat(decode_e4m3(s), 16, axis=1)


def make_problem(E, N, K, counts, seed, a_scale=1.0):
    torch.manual_seed(seed)
    lay, rows = host_layout(counts, np.ones(E, np.int64))
    rows = max(rows, 128)
    A = (torch.randn(rows, K, device="cuda") * a_scale).to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
    ac, asf = quantize_nvfp4(A)
    wc, wsf = quantize_nvfp4(W)
    return lay, rows, A, W, ac, asf, wc, wsf


@pytest.fixture(params=["1", "2", "v2"], ids=["cta1", "pair", "pair_a_resident"])
def cluster(request, monkeypatch):
    """Every kernel form: v1 with one CTA per tile, v1 with 2-CTA pairs (cta_group::2,
    M = 256, odd m-tile counts give the rank-1 CTA a dummy slot), and the v2 STORE
    kernel (gemm_fp4_pair.cu: pairs, A resident, N = 128 double-buffered; the default
    for STORE with K <= 1536, other shapes fall back to v1)."""
    if request.param == "v2":
        monkeypatch.delenv("REALB_GEMM_CLUSTER", raising=False)
        monkeypatch.setenv("REALB_K6_VERSION", "2")
    else:
        monkeypatch.setenv("REALB_GEMM_CLUSTER", request.param)
        monkeypatch.setenv("REALB_K6_VERSION", "1")
    return request.param


@pytest.mark.parametrize("E,N,K,counts", [
    (1, 256, 256, [128]),
    (3, 512, 1408, [1500, 700, 2100]),       # pair units with odd and even m-tile counts
    (1, 256, 64, [100]),
    (3, 512, 2048, [300, 0, 700]),
    (4, 2048, 1408, [513, 129, 1, 260]),     # Kimi down: K tail (1408 = 5.5 x 256)
    (4, 2816, 2048, [513, 129, 1, 260]),     # Kimi gate_up
])
def test_fp4_store_vs_dequant_oracle(E, N, K, counts, cluster, parity_log):
    lay, rows, A, W, ac, asf, wc, wsf = make_problem(E, N, K, counts, seed=E + N + K)
    out = torch.full((rows, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    lt = torch.from_numpy(lay).cuda()
    _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
              rows, N, K, E, lt.data_ptr(), _lib.EPI_STORE, out.data_ptr(), None, None, 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    Ad = dequant(ac, asf, rows, K)
    Wd = dequant(wc, wsf, E * N, K)
    for e in range(E):
        if counts[e] == 0:
            continue
        rs = int(lay[8 + e])
        ref = Ad[rs:rs + counts[e]] @ Wd[e * N:(e + 1) * N].T
        got = out[rs:rs + counts[e]].float().cpu().numpy()
        # vs the exact product of the dequantised operands rounded to bf16 (the kernel's
        # one output rounding): fp32 accumulation order is all that remains
        refb = bf16_round(ref.astype(np.float32))
        err = np.linalg.norm(got - refb) / np.linalg.norm(refb)
        parity_log("k6_vs_dequant_oracle_bf16_rounded", err, 1e-3)
        assert err < 1e-3, (e, err)


@pytest.mark.parametrize("counts", [[200, 77], [1100, 390]])
def test_fp4_swiglu_requant_epilogue(counts, cluster, parity_log):
    """K4 fused into K6's SwiGLU epilogue, bit-exact: the NVFP4 codes and scales
    the kernel writes equal the reference block rule (oracle, fp4.py:173-227)
    applied to the bf16 SwiGLU values the kernel itself computed (read back
    through the d_out parity hook). Those bf16 values in turn match the oracle's
    fp32 SwiGLU of the dequantised GEMM within bf16 rounding."""
    E, N, K = 2, 512, 512
    lay, rows, A, W, ac, asf, wc, wsf = make_problem(E, N, K, counts, seed=5, a_scale=4.0)
    I = N // 2
    hc = torch.zeros(rows, I // 2, dtype=torch.uint8, device="cuda")
    hsf = torch.zeros(rows * I // 16, dtype=torch.uint8, device="cuda")
    hbf = torch.zeros(rows, I, dtype=torch.bfloat16, device="cuda")
    lt = torch.from_numpy(lay).cuda()
    _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
              rows, N, K, E, lt.data_ptr(), _lib.EPI_SWIGLU, hbf.data_ptr(), hc.data_ptr(), hsf.data_ptr(), 0,
              _lib.stream_ptr())
    torch.cuda.synchronize()
    Ad = dequant(ac, asf, rows, K)
    Wd = dequant(wc, wsf, E * N, K)
    hc_np = hc.cpu().numpy()
    hsf_flat = sf_mma_to_flat(hsf.cpu().numpy(), rows, I)
    hbits = hbf.view(torch.int16).cpu().numpy().view(np.uint16)
    from oracle.moe_ref import bf16_round, silu

    for e in range(E):
        rs = int(lay[8 + e])
        sl = slice(rs, rs + counts[e])
        # exact: the kernel's codes / scales == the reference rule on the kernel's own bf16 h
        oc, osf = oracle.quantize_bf16(hbits[sl])
        assert (hc_np[sl] == oc).all()
        assert (hsf_flat[sl] == osf).all()
        # the bf16 h itself vs the oracle's SwiGLU (fp32 accumulation order, __expf)
        y = Ad[sl] @ Wd[e * N:(e + 1) * N].T          # interleaved halves
        y = y.reshape(counts[e], N // 256, 2, 128)
        h = bf16_round((silu(y[:, :, 0]) * y[:, :, 1]).reshape(counts[e], I).astype(np.float32))
        got = hbf[sl].float().cpu().numpy()
        err = np.linalg.norm(got - h) / np.linalg.norm(h)
        parity_log("k6_swiglu_h_vs_oracle", err, 2e-3)
        assert err < 2e-3, err


def _scatter_map(lay, counts, n_dst, seed):
    """A random row map over the valid rows: row g -> (destination d, row j), each
    destination's rows a permutation of 0..n_d-1."""
    rng = np.random.default_rng(seed)
    valid = np.concatenate([int(lay[8 + e]) + np.arange(c) for e, c in enumerate(counts)]).astype(np.int64)
    d = rng.integers(0, n_dst, len(valid))
    rowmap = {}
    sizes = []
    for dd in range(n_dst):
        sel = valid[d == dd]
        perm = rng.permutation(len(sel))
        for g, j in zip(sel, perm):
            rowmap[int(g)] = (dd, int(j))
        sizes.append(len(sel))
    return rowmap, sizes


@pytest.mark.parametrize("E,N,K,counts,n_dst", [
    (3, 512, 1408, [300, 0, 700], 2),
    (4, 2048, 1408, [513, 129, 1, 260], 5),     # Kimi down
])
def test_fp4_scatter_equals_store(E, N, K, counts, n_dst):
    """realb_grouped_gemm_nvfp4_scatter: every valid row lands, bit-identical to
    the STORE epilogue's row, at its mapped (destination, row); nothing else is
    written."""
    lay, rows, A, W, ac, asf, wc, wsf = make_problem(E, N, K, counts, seed=7 + E)
    lay_t = torch.from_numpy(lay).cuda()
    ref = torch.zeros((rows, N), dtype=torch.bfloat16, device="cuda")
    _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(), rows, N, K,
              E, lay_t.data_ptr(), _lib.EPI_STORE, ref.data_ptr(), None, None, 0, _lib.stream_ptr())
    rowmap, sizes = _scatter_map(lay, counts, n_dst, seed=E)
    m = np.full(rows, -1, np.int32)
    for g, (d, j) in rowmap.items():
        m[g] = (d << 25) | j
    m_t = torch.from_numpy(m).cuda()
    dsts = [torch.full((max(s, 1) + 1, N), 7.0, dtype=torch.bfloat16, device="cuda") for s in sizes]
    bases = np.array([t.data_ptr() for t in dsts], np.uint64)
    _lib.call("realb_grouped_gemm_nvfp4_scatter", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
              rows, N, K, E, lay_t.data_ptr(), m_t.data_ptr(), n_dst, bases.ctypes.data, 0, _lib.stream_ptr())
    torch.cuda.synchronize()
    got = [t.cpu() for t in dsts]
    refc = ref.cpu()
    for g, (d, j) in rowmap.items():
        assert torch.equal(got[d][j], refc[g]), (g, d, j)
    for d, s in enumerate(sizes):
        assert (got[d][s:].float() == 7.0).all()


@pytest.mark.parametrize("E,N,K,counts,epi", [
    (8, 2048, 1408, None, "store"),             # Kimi EP8 hot rank, down GEMM
    (8, 2816, 2048, None, "swiglu"),            # Kimi EP8 hot rank, gate_up GEMM (+ K4 epilogue)
    (5, 512, 768, [1, 0, 383, 129, 1000], "store"),   # Qwen down K, odd / empty / 1-row experts
    (5, 1536, 2048, [1, 0, 383, 129, 1000], "swiglu"),  # Qwen gate_up
    (2, 2560, 512, [700, 300], "store"),        # ERNIE-vision down K
    (3, 1024, 1024, [256, 255, 257], "swiglu"),
])
def test_fp4_v2_equals_v1(E, N, K, counts, epi, monkeypatch):
    """K6 v2 (pair, A resident) and v1 (1-CTA) give bit-identical outputs (bf16 for
    STORE; NVFP4 codes, scales and the bf16 SwiGLU hook for SWIGLU): the same K=64
    block-scaled MMAs in the same k order; only tiling and feed differ."""
    if counts is None:
        counts = ((np.random.default_rng(0).random(E) * 0.2 + 0.9) * 17134).astype(np.int64).tolist()
    lay, rows, A, W, ac, asf, wc, wsf = make_problem(E, N, K, counts, seed=7 + K)
    lt = torch.from_numpy(lay).cuda()
    outs = []
    monkeypatch.delenv("REALB_GEMM_CLUSTER", raising=False)
    for ver in ("1", "2", "2"):  # v2 twice: the tile counters re-arm between launches
        monkeypatch.setenv("REALB_K6_VERSION", ver)
        if epi == "store":
            out = torch.full((rows, N), float("nan"), dtype=torch.bfloat16, device="cuda")
            _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
                      rows, N, K, E, lt.data_ptr(), _lib.EPI_STORE, out.data_ptr(), None, None, 0,
                      _lib.stream_ptr())
            res = [out.view(torch.int16)]
        else:
            I = N // 2
            hc = torch.zeros(rows, I // 2, dtype=torch.uint8, device="cuda")
            hsf = torch.zeros(rows * I // 16, dtype=torch.uint8, device="cuda")
            hbf = torch.zeros(rows, I, dtype=torch.bfloat16, device="cuda")
            _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
                      rows, N, K, E, lt.data_ptr(), _lib.EPI_SWIGLU, hbf.data_ptr(), hc.data_ptr(), hsf.data_ptr(),
                      0, _lib.stream_ptr())
            res = [hbf.view(torch.int16), hc, hsf]  # scales: MMA layout, compared whole
        torch.cuda.synchronize()
        outs.append(res)
    valid = torch.zeros(rows, dtype=torch.bool)
    for e in range(E):
        rs = int(lay[8 + e])
        valid[rs:rs + counts[e]] = True
    valid = valid.cuda()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            if a.dim() == 1:
                assert torch.equal(a, b), int((a != b).sum())
            else:
                assert torch.equal(a[valid], b[valid]), int((a[valid] != b[valid]).sum())
