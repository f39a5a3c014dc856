"""Pin the CPU oracle (oracle/fp4_oracle.c) to the reference before trusting it.

Fixtures come from running the reference itself (tests/golden/make_golden.py);
the golden file SHA-256 is the reference's own (tests/test_fp4.py:194-210)."""

import hashlib
import json

import numpy as np
import pytest

import gen
import oracle


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_regimes_match_reference_fixture(golden):
    d = np.load(golden / "fp4_regimes.npz")
    c, s = oracle.quantize_blocks(d["values"])
    assert (c == d["codes"]).all() and (s == d["scale_bits"]).all()


def test_all_bf16_amax_scales(golden):
    s_ref = np.load(golden / "fp4_bf16_amax.npz")["scale_bits"]
    _, s = oracle.quantize_blocks(gen.bf16_amax_blocks())
    assert (s == s_ref).all()


def test_exhaustive_bf16_code_table(golden):
    dig = json.loads((golden / "fp4_digests.json").read_text())
    blocks = gen.bf16_code_table_blocks()
    assert len(blocks) == dig["code_table"]["blocks"]
    assert _digest(*oracle.quantize_blocks(blocks)) == dig["code_table"]["sha256"]


def test_acceptance_criterion_9_digest(golden):
    dig = json.loads((golden / "fp4_digests.json").read_text())
    c, s = oracle.quantize_blocks(gen.acceptance_blocks())
    assert _digest(c, s) == dig["acceptance_909"]["sha256"]


def test_golden_file_sha256(tmp_path):
    from paper_2604_19503_b200.quant import write_blocks

    vals = np.array(gen.GOLDEN_FILE_INPUT).reshape(-1, 16)
    c, s = oracle.quantize_blocks(vals)
    p = tmp_path / "g.fp4"
    write_blocks(c, s, 32, p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == gen.GOLDEN_FILE_SHA256


def test_reference_known_answers():
    # tests/test_fp4.py:40-44 (E4M3 ties) and :58-64 (E2M1 ties), via whole blocks
    def q(vals):
        c, s = oracle.quantize_blocks(np.array([vals], float))
        return oracle.dequantize_blocks(c, s)[0]

    for v, exp in [(0.25, 0.0), (0.75, 1.0), (1.25, 1.0), (1.75, 2.0), (2.5, 2.0), (3.5, 4.0), (5.0, 4.0)]:
        out = q([6.0, v, -v] + [0.0] * 13)
        assert out[1] == exp and out[2] == -exp
    # amax/6 = 1.0625 -> scale 1.0 ; 1.1875 -> 1.25
    assert oracle.quantize_blocks(np.array([[6 * 1.0625] + [0.0] * 15]))[1][0] == 0x38
    assert oracle.quantize_blocks(np.array([[6 * 1.1875] + [0.0] * 15]))[1][0] == 0x3A
    with pytest.raises(oracle.OracleDomainError):
        oracle.quantize_blocks(np.array([[np.nan] + [0.0] * 15]))


def test_bf16_fast_path_matches_block_rule():
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((64, 256)) * 0.02).astype(np.float32)
    bits = (x.view(np.uint32) >> 16).astype(np.uint16)
    xb = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    codes, sf = oracle.quantize_bf16(bits)
    c2, s2 = oracle.quantize_blocks(xb.reshape(-1, 16))
    from paper_2604_19503_b200.quant import unpack_codes

    assert (unpack_codes(codes).reshape(-1, 16) == c2).all()
    assert (sf.reshape(-1) == s2).all()


def test_oracle_against_live_reference(reference):
    rng = np.random.default_rng(123)
    vals = rng.normal(0, 1, (3000, 16)) * np.exp2(rng.integers(-30, 14, (3000, 1)).astype(float))
    from moesim.fp4 import quantize_blocks as ref_q

    c_ref, s_ref = ref_q(vals)
    c, s = oracle.quantize_blocks(vals)
    assert (c == c_ref).all() and (s == s_ref).all()
