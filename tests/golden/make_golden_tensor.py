"""Generate tests/golden/fp4_tensor_cases.npz by running the REFERENCE's
quantize_tensor + ErrorSummary and pack_block (moesim/fp4.py:137-170, :246-252)
on gen.tensor_cases(). Run in the build container:
    python tests/golden/make_golden_tensor.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import gen  # noqa: E402
from moesim.fp4 import pack_block, quantize_tensor  # noqa: E402


def main():
    out = {}
    for i, v in enumerate(gen.tensor_cases()):
        blocks, summ = quantize_tensor([float(a) for a in v])
        out[f"c{i}_values"] = v
        out[f"c{i}_records"] = np.frombuffer(b"".join(pack_block(b) for b in blocks), np.uint8).reshape(-1, 9)
        out[f"c{i}_rmse"] = np.float64(summ.rmse)
        out[f"c{i}_rel_rmse"] = np.float64(summ.relative_rmse)
        out[f"c{i}_max_rel"] = np.array(summ.max_relative_error_per_block, np.float64)
    np.savez_compressed(HERE / "fp4_tensor_cases.npz", n=len(gen.tensor_cases()), **out)
    print("cases:", len(gen.tensor_cases()))


if __name__ == "__main__":
    main()
