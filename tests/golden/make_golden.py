"""Generate the committed golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures are small (<1 MB); large exhaustive outputs are committed as
SHA-256 digests of the reference's output arrays and regenerated inputs
(tests/golden/gen.py) are checked against them.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import gen  # noqa: E402
from moesim import (  # noqa: E402
    ClusterConfig,
    RankLoad,
    RealbParams,
    plan_realb,
)
from moesim.fp4 import quantize_blocks, quantize_tensor, write_blocks  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {}
    # 1. regimes (full arrays)
    vals = gen.fp4_regime_blocks()
    c, s = quantize_blocks(vals)
    np.savez_compressed(HERE / "fp4_regimes.npz", values=vals, codes=c, scale_bits=s)
    # 2. all bf16 amax -> scale bits (full array)
    amax = gen.bf16_amax_blocks()
    _, s_amax = quantize_blocks(amax)
    np.savez_compressed(HERE / "fp4_bf16_amax.npz", scale_bits=s_amax)
    # 3. digests of the large exhaustive / acceptance sets
    ct = gen.bf16_code_table_blocks()
    c_ct, s_ct = quantize_blocks(ct)
    out["code_table"] = {"blocks": int(len(ct)), "sha256": digest(c_ct, s_ct)}
    acc = gen.acceptance_blocks()
    c_acc, s_acc = quantize_blocks(acc)
    out["acceptance_909"] = {"blocks": int(len(acc)), "sha256": digest(c_acc, s_acc)}
    # 4. golden file bytes (tests/test_fp4.py:194-210)
    blocks, _ = quantize_tensor(gen.GOLDEN_FILE_INPUT)
    p = Path("/tmp/_golden.fp4")
    write_blocks(blocks, 32, p)
    out["golden_file_sha256"] = hashlib.sha256(p.read_bytes()).hexdigest()
    assert out["golden_file_sha256"] == gen.GOLDEN_FILE_SHA256
    (HERE / "fp4_digests.json").write_text(json.dumps(out, indent=1) + "\n")

    # 5. policy cases
    cases = gen.policy_cases()
    for cs in cases:
        R = len(cs["v"])
        loads = [RankLoad(r, cs["v"][r], cs["t"][r]) for r in range(R)]
        cfg = ClusterConfig(num_ranks=R, num_layers=1, experts_per_rank=1, bytes_per_expert=1,
                            modality_isolated=cs["iso"])
        plan = plan_realb(loads, RealbParams(cs["C"], cs["Md"], cs["thr"]), cfg)
        cs["expect"] = {
            "prec": [p.value for p in plan.per_rank_precision],
            "hot": sorted(plan.hot_ranks),
            "vision": sorted(plan.vision_heavy_ranks),
            "active": plan.active,
        }
    (HERE / "policy_cases.json").write_text(json.dumps(cases) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
