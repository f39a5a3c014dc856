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


# ---- oracle/fp4_numpy.py (the "reference quantiser" CPU baseline bench.py times)
def test_numpy_quantiser_matches_reference_fixtures(golden):
    from oracle import fp4_numpy

    d = np.load(golden / "fp4_regimes.npz")
    c, s = fp4_numpy.quantize_blocks(d["values"])
    assert (c == d["codes"]).all() and (s == d["scale_bits"]).all()
    s_ref = np.load(golden / "fp4_bf16_amax.npz")["scale_bits"]
    assert (fp4_numpy.quantize_blocks(gen.bf16_amax_blocks())[1] == s_ref).all()
    dig = json.loads((golden / "fp4_digests.json").read_text())
    assert _digest(*fp4_numpy.quantize_blocks(gen.acceptance_blocks())) == dig["acceptance_909"]["sha256"]
    with pytest.raises(ValueError):
        fp4_numpy.quantize_blocks(np.array([[np.inf] + [0.0] * 15]))


def test_numpy_quantiser_exhaustive_code_table(golden):
    from oracle import fp4_numpy

    dig = json.loads((golden / "fp4_digests.json").read_text())
    assert _digest(*fp4_numpy.quantize_blocks(gen.bf16_code_table_blocks())) == dig["code_table"]["sha256"]


# ---- oracle/policy_ref.py (the CPU arms' policy, independent of the product library)
def test_policy_ref_matches_reference_fixture(golden):
    from oracle import policy_ref

    for cs in json.loads((golden / "policy_cases.json").read_text()):
        R = len(cs["v"])
        p = policy_ref.plan_realb([(r, cs["v"][r], cs["t"][r]) for r in range(R)], cs["C"], cs["Md"], cs["thr"],
                                  cs["iso"])
        e = cs["expect"]
        assert ["w4a4" if x else "w16a16" for x in p["precision"]] == e["prec"], cs
        assert sorted(p["hot"]) == e["hot"] and sorted(p["vision"]) == e["vision"] and p["active"] == e["active"]


def test_policy_ref_fuzz_against_live_reference(reference):
    from moesim import ClusterConfig as RC, ExpertPlacement as RP, RankLoad as RL, RealbParams as RPar
    from moesim import aggregate_rank_loads as ragg, plan_realb as rplan

    from oracle import policy_ref

    rng = np.random.default_rng(31)
    for _ in range(500):
        R = int(rng.choice([2, 3, 4, 8]))
        epr = int(rng.choice([1, 2, 4]))
        E = R * epr
        hosts = [(e // epr,) + ((int(rng.integers(0, R)),) if rng.random() < 0.2 else ()) for e in range(E)]
        hosts = [tuple(dict.fromkeys(h)) for h in hosts]
        loads = {e: (int(rng.integers(0, 900)), int(rng.integers(0, 900))) for e in range(E) if rng.random() < 0.9}
        place = RP(assignment=tuple(hosts), redundant_count=sum(len(h) - 1 for h in hosts))
        rl = ragg(loads, place, R)
        ol = policy_ref.aggregate_rank_loads(loads, hosts, R)
        assert [(l.rank, l.vision_tokens, l.text_tokens) for l in rl] == ol
        if rng.random() < 0.3:  # out-of-order rank ids
            perm = rng.permutation(R)
            rl, ol = [rl[i] for i in perm], [ol[i] for i in perm]
        C, Md, thr, iso = float(rng.choice([0.5, 1.0, 1.3])), float(rng.random()), int(rng.choice([0, 2048])), \
            bool(rng.random() < 0.3)
        ref = rplan(rl, RPar(C, Md, thr), RC(R, 1, epr, 1, iso))
        got = policy_ref.plan_realb(ol, C, Md, thr, iso)
        assert got["precision"] == [int(p.value == "w4a4") for p in ref.per_rank_precision]
        assert got["hot"] == ref.hot_ranks and got["vision"] == ref.vision_heavy_ranks and got["active"] == ref.active


def test_quantize_tensor_oracle_matches_reference_fixture(golden):
    """oracle.quantize_tensor == the reference's quantize_tensor + ErrorSummary +
    pack_block on every fixture case, bit for bit (sums in the reference's order)."""
    d = np.load(golden / "fp4_tensor_cases.npz")
    for i in range(int(d["n"])):
        rec, rmse, rel, mr = oracle.quantize_tensor(d[f"c{i}_values"])
        assert (rec == d[f"c{i}_records"]).all(), i
        assert rmse == float(d[f"c{i}_rmse"]) and rel == float(d[f"c{i}_rel_rmse"]), i
        assert (mr == d[f"c{i}_max_rel"]).all(), i


def test_read_write_blocks_interoperate_with_reference(reference, tmp_path):
    """Q6: our write_blocks / read_blocks / unpack_block / pack_block (host byte
    format) against the reference's, both directions."""
    from moesim import fp4 as rf

    from paper_2604_19503_b200 import quant

    vals = list(gen.GOLDEN_FILE_INPUT) + [0.3, -7.0, 1e-5]
    rblocks, _ = rf.quantize_tensor(vals)
    p1 = tmp_path / "ref.fp4"
    rf.write_blocks(rblocks, len(vals), p1)
    ours, count = quant.read_blocks(p1)
    assert count == len(vals)
    assert [(b.codes, b.scale_bits) for b in ours] == [(b.codes, b.scale_bits) for b in rblocks]
    p2 = tmp_path / "ours.fp4"
    quant.write_blocks(ours, len(vals), p2)
    assert p2.read_bytes() == p1.read_bytes()
    back, c2 = rf.read_blocks(p2)
    assert c2 == len(vals) and back == rblocks
    for rb in rblocks:
        assert quant.pack_block(quant.Fp4Block(rb.codes, rb.scale_bits)) == rf.pack_block(rb)
        assert quant.unpack_block(rf.pack_block(rb)).codes == rb.codes
    with pytest.raises(ValueError):
        quant.unpack_block(b"\x00" * 8)
    bad = tmp_path / "bad.fp4"
    bad.write_bytes(b"FP4REF02" + p1.read_bytes()[8:])
    with pytest.raises(ValueError, match="magic"):
        quant.read_blocks(bad)
    bad.write_bytes(p1.read_bytes()[:-1])
    with pytest.raises(ValueError, match="truncated"):
        quant.read_blocks(bad)
    with pytest.raises(ValueError):
        quant.Fp4Block((0,) * 15, 0)
    with pytest.raises(ValueError):
        quant.Fp4Block((16,) + (0,) * 15, 0)
    with pytest.raises(ValueError):
        quant.Fp4Block((0,) * 16, 0x80)
