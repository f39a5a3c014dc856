"""K3 parity on the GPU: the CUDA quantiser vs the pinned oracle / reference
fixtures, bit-exact, plus the MMA scale layout and the domain-error path."""

import hashlib
import json

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def q():
    from paper_2604_19503_b200 import quant

    return quant


def test_regimes_bit_exact(q, golden):
    d = np.load(golden / "fp4_regimes.npz")
    c, s = q.quantize_blocks(d["values"])
    assert (c == d["codes"]).all() and (s == d["scale_bits"]).all()


def test_all_bf16_amax(q, golden):
    s_ref = np.load(golden / "fp4_bf16_amax.npz")["scale_bits"]
    _, s = q.quantize_blocks(gen.bf16_amax_blocks())
    assert (s == s_ref).all()


@pytest.mark.parametrize("dtype", ["float64", "float32", "bfloat16"])
def test_exhaustive_code_table(q, golden, dtype):
    import torch

    dig = json.loads((golden / "fp4_digests.json").read_text())["code_table"]
    blocks = gen.bf16_code_table_blocks()  # every value is a bf16 value: exact in all dtypes
    t = torch.from_numpy(blocks).to(getattr(torch, dtype))
    c, s = q.quantize_blocks(t)
    assert _digest(c, s) == dig["sha256"]


def test_acceptance_1e6_blocks(q, golden):
    dig = json.loads((golden / "fp4_digests.json").read_text())["acceptance_909"]
    c, s = q.quantize_blocks(gen.acceptance_blocks())
    assert _digest(c, s) == dig["sha256"]


def test_golden_file_from_gpu_codes(q, tmp_path):
    c, s = q.quantize_blocks(np.array(gen.GOLDEN_FILE_INPUT).reshape(-1, 16))
    p = tmp_path / "g.fp4"
    q.write_blocks(c, s, 32, p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == gen.GOLDEN_FILE_SHA256


def test_nonfinite_raises(q):
    for bad in (np.inf, -np.inf, np.nan):
        v = np.zeros((3, 16))
        v[1, 5] = bad
        with pytest.raises(q.QuantizationDomainError):
            q.quantize_blocks(v)


@pytest.mark.parametrize("rows,cols", [(128, 64), (256, 2048), (2816, 2048), (2048, 1408), (384, 192)])
def test_bf16_weights_mma_layout(q, rows, cols):
    """Product path: bf16 weight matrix -> packed codes + MMA scale layout, vs the
    oracle on the same bf16 values (N(0, 0.02): the subnormal-scale regime)."""
    import torch

    g = torch.Generator(device="cpu").manual_seed(rows * 7 + cols)
    w = (torch.randn(rows, cols, generator=g) * 0.02).to(torch.bfloat16)
    codes, sf = q.quantize_nvfp4(w.cuda(), layout="mma")
    codes_f, sf_f = q.quantize_nvfp4(w.cuda(), layout="flat")
    bits = w.view(torch.int16).numpy().view(np.uint16)
    oc, osf = oracle.quantize_bf16(bits)
    assert (codes.cpu().numpy() == oc).all()
    assert (codes_f.cpu().numpy() == oc).all()
    assert (sf_f.cpu().numpy() == osf).all()
    assert (q.sf_mma_to_flat(sf.cpu().numpy(), rows, cols) == osf).all()


def test_mma_layout_matches_torch_to_blocked(q):
    """Third-party cross-check of the scale layout: torch's cuBLAS 'to_blocked'
    (torch/testing/_internal/common_quantized.py) on the flat scales."""
    import torch

    rows, cols = 256, 512
    w = (torch.randn(rows, cols) * 3).to(torch.bfloat16).cuda()
    _, sf = q.quantize_nvfp4(w, layout="mma")
    _, sf_f = q.quantize_nvfp4(w, layout="flat")
    m = sf_f.view(rows, cols // 16)
    n_rb, n_cb = rows // 128, cols // 64
    blocked = m.view(n_rb, 128, n_cb, 4).permute(0, 2, 1, 3).reshape(-1, 4, 32, 4).transpose(1, 2)
    assert torch.equal(blocked.reshape(-1), sf.view(-1))


def test_max_ctas_and_stream(q):
    import torch

    w = torch.randn(1024, 2048, dtype=torch.bfloat16, device="cuda")
    ref = q.quantize_nvfp4(w)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = q.quantize_nvfp4(w, max_ctas=16, stream=s)
    s.synchronize()
    assert torch.equal(ref[0], out[0]) and torch.equal(ref[1], out[1])


def test_all_bf16_amax_bf16_path(q, golden):
    """Every positive finite bf16 amax through the bf16 product path (the
    division-free scale computation), vs the reference's scale bits."""
    import torch

    s_ref = np.load(golden / "fp4_bf16_amax.npz")["scale_bits"]
    blocks = torch.from_numpy(gen.bf16_amax_blocks()).to(torch.bfloat16)
    _, s = q.quantize_blocks(blocks)
    assert (s == s_ref).all()


def test_bf16_path_row_tail_and_flat_layout(q):
    """Rows not a multiple of 128 and the 64-row pairing of the tile routine."""
    import torch

    for rows, cols in [(1, 16), (63, 48), (65, 64), (130, 208), (191, 1408)]:
        w = (torch.randn(rows, cols) * 3).to(torch.bfloat16)
        codes, sf = q.quantize_nvfp4(w.cuda(), layout="flat")
        oc, osf = oracle.quantize_bf16(w.view(torch.int16).numpy().view(np.uint16))
        assert (codes.cpu().numpy() == oc).all() and (sf.cpu().numpy() == osf).all(), (rows, cols)


# ---------------------------------------------------------------- Q5 / Q6 on the device
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_quantize_tensor_vs_reference_fixture(q, golden, dtype, parity_log):
    """realb_quantize_tensor_nvfp4 == the reference's quantize_tensor +
    ErrorSummary + pack_block (fixture from the reference itself): block records
    and per-block max relative errors bit-exact; rmse / relative rmse within
    1e-12 (device tree-order sums vs the reference's sequential sums)."""
    import torch

    d = np.load(golden / "fp4_tensor_cases.npz")
    for i in range(int(d["n"])):
        v = d[f"c{i}_values"]
        if dtype == "f32" and not (v.astype(np.float32).astype(np.float64) == v).all():
            continue  # f32 input must hold the same values
        t = torch.from_numpy(v.astype(np.float64 if dtype == "f64" else np.float32)).cuda()
        r = q.quantize_tensor_device(t)
        torch.cuda.synchronize()
        assert int(r["flag"].item()) == 0
        assert (r["records"].cpu().numpy() == d[f"c{i}_records"]).all(), i
        assert (r["max_rel"].cpu().numpy() == d[f"c{i}_max_rel"]).all(), i
        s = q.summary_from_sums(r["sums"], r["n"])
        for got, ref in ((s.rmse, float(d[f"c{i}_rmse"])), (s.relative_rmse, float(d[f"c{i}_rel_rmse"]))):
            assert abs(got - ref) <= 1e-12 * max(abs(ref), 1e-300), (i, got, ref)
            parity_log("quantize_tensor_rmse_rel_diff", abs(got - ref) / max(abs(ref), 1e-300), 1e-12)


def test_quantize_tensor_reference_api(q, golden, tmp_path):
    """The reference-shaped API (list in -> (list[Fp4Block], ErrorSummary)), its
    error behaviour, the reference test cases (tests/test_fp4.py:151-179) and the
    golden file written from device-produced blocks."""
    import math

    blocks, s = q.quantize_tensor(gen.ON_GRID)
    assert s.rmse == 0.0
    blocks, s = q.quantize_tensor([6.0] * 17)
    assert len(blocks) == 2 and s.rmse == 0.0 and s.max_relative_error_per_block == (0.0, 0.0)
    _, s = q.quantize_tensor([6.0] * 16 + [1.25])
    tail = q.dequantize_block(q.quantize_tensor([1.25])[0][0])[0]
    assert s.rmse == math.sqrt((1.25 - tail) ** 2 / 17)
    _, s = q.quantize_tensor(list(map(float, np.random.default_rng(0).standard_normal(4096))))
    assert s.relative_rmse < 0.10
    with pytest.raises(ValueError):
        q.quantize_tensor([])
    with pytest.raises(ValueError):
        q.quantize_tensor([1.0] * 16, block_size=32)
    with pytest.raises(q.QuantizationDomainError):
        q.quantize_tensor([1.0, float("nan")])
    blocks, _ = q.quantize_tensor(gen.GOLDEN_FILE_INPUT)
    p = tmp_path / "g.fp4"
    q.write_blocks(blocks, 32, p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == gen.GOLDEN_FILE_SHA256
    back, count = q.read_blocks(p)
    assert count == 32 and back == blocks
    assert q.quantize_block(gen.ON_GRID) == blocks[0]
    assert q.dequantize_block(blocks[0]) == gen.ON_GRID
    assert blocks[0].scale == 1.0


def test_dequantize_blocks_vs_oracle(q, golden):
    d = np.load(golden / "fp4_regimes.npz")
    got = q.dequantize_blocks(d["codes"], d["scale_bits"])
    assert (got == oracle.dequantize_blocks(d["codes"], d["scale_bits"])).all()
    # every (code, scale) pattern, including 0x7F (decodes to 480, fp4.py:59-66)
    codes = np.tile(np.arange(16, dtype=np.uint8), (128, 1))
    sb = np.arange(128, dtype=np.uint8)
    assert (q.dequantize_blocks(codes, sb) == oracle.dequantize_blocks(codes, sb)).all()


def test_weight_error_summary_bf16_weights(q):
    """The accuracy proxy the bench reports for W4A4 ranks: bf16 N(0, 0.02) weights
    through the device summary == the oracle's quantize_tensor on the same values."""
    import torch

    w = (torch.randn(256, 1408, generator=torch.Generator().manual_seed(4)) * 0.02).to(torch.bfloat16)
    r = q.quantize_tensor_device(w.cuda())
    torch.cuda.synchronize()
    rec, rmse, rel, mr = oracle.quantize_tensor(w.float().numpy().astype(np.float64).reshape(-1))
    assert (r["records"].cpu().numpy() == rec).all()
    assert (r["max_rel"].cpu().numpy() == mr).all()
    s = q.summary_from_sums(r["sums"], r["n"])
    assert abs(s.relative_rmse - rel) <= 1e-12 * rel and abs(s.rmse - rmse) <= 1e-12 * rmse
    assert 0.09 < s.relative_rmse < 0.12  # subnormal-scale regime (0.103)


@pytest.mark.parametrize("max_ctas", [0, 7])
def test_experts2_one_launch_bit_exact(q, max_ctas):
    """realb_quantize_experts2_nvfp4: an expert set's gate_up [E*2I, H] and down
    [E*H, I] weights in ONE launch (the tile range crosses from one matrix to the
    other inside CTAs) == the oracle on each W4A4 expert's rows; W16A16 experts'
    outputs untouched. Kimi-like I = 1408 (22 k-tiles) next to H = 2048 (32)."""
    import torch
    from paper_2604_19503_b200 import _lib

    E, H, I = 5, 256, 1408
    g = torch.Generator(device="cpu").manual_seed(11)
    wgu = (torch.randn(E * 2 * I, H, generator=g) * 0.02).to(torch.bfloat16)
    wd = (torch.randn(E * H, I, generator=g) * 0.02).to(torch.bfloat16)
    prec = np.array([1, 0, 1, 1, 0], np.uint8)
    dev = {k: v.cuda() for k, v in dict(wgu=wgu, wd=wd).items()}
    cg = torch.full((E * 2 * I, H // 2), 0xAB, dtype=torch.uint8, device="cuda")
    sg = torch.full((E * 2 * I * H // 16,), 0xAB, dtype=torch.uint8, device="cuda")
    cd = torch.full((E * H, I // 2), 0xAB, dtype=torch.uint8, device="cuda")
    sd = torch.full((E * H * I // 16,), 0xAB, dtype=torch.uint8, device="cuda")
    pd = torch.from_numpy(prec).cuda()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("realb_quantize_experts2_nvfp4", dev["wgu"].data_ptr(), 2 * I, H, cg.data_ptr(), sg.data_ptr(),
              dev["wd"].data_ptr(), H, I, cd.data_ptr(), sd.data_ptr(), E, pd.data_ptr(), flag.data_ptr(),
              max_ctas, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    for w, c, sfm, rpe, cols in ((wgu, cg, sg, 2 * I, H), (wd, cd, sd, H, I)):
        c = c.cpu().numpy()
        sfm = sfm.cpu().numpy().reshape(E, -1)
        for e in range(E):
            rows = slice(e * rpe, (e + 1) * rpe)
            if prec[e]:
                bits = w[rows].view(torch.int16).numpy().view(np.uint16)
                oc, osf = oracle.quantize_bf16(bits)
                assert (c[rows] == oc).all()
                assert (q.sf_mma_to_flat(sfm[e], rpe, cols) == osf).all()
            else:
                assert (c[rows] == 0xAB).all() and (sfm[e] == 0xAB).all()
