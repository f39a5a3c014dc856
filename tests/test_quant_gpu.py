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
