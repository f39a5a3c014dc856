"""The compile-time table of E4M3 scale reciprocals in fp4_rule.cuh (read by the
activation-side block rule: K4 producers and the K6 SwiGLU re-quantisation) holds the
correctly rounded fp32 reciprocal of every nonzero scale code, i.e. what __frcp_rn
returns: built from the header with nvcc's constant evaluator, compared with numpy's
IEEE float32 division. CPU-only (compiles a host program)."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2604_19503_b200" / "csrc"

PROG = r'''
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include "fp4_rule.cuh"
int main() {
  constexpr realb::E4M3Rcp t = realb::make_e4m3_rcp();
  for (unsigned b = 1; b < 128; ++b) {
    unsigned r, s;
    const float sc = realb::e4m3_decode_ce(b);
    std::memcpy(&r, &t.v[b], 4);
    std::memcpy(&s, &sc, 4);
    std::printf("%u %08x %08x\n", b, s, r);
  }
  return 0;
}
'''


def _nvcc():
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and Path(c).exists():
            return c
    return None


@pytest.mark.skipif(_nvcc() is None, reason="nvcc not available")
def test_compile_time_reciprocals_are_ieee(tmp_path):
    src = tmp_path / "rcp.cu"
    src.write_text(PROG)
    exe = tmp_path / "rcp"
    subprocess.run([_nvcc(), "-std=c++17", "-I", str(CSRC), str(src), "-o", str(exe)], check=True,
                   capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    rows = [line.split() for line in out if line.strip()]
    assert len(rows) == 127
    for b, sbits, rbits in rows:
        sc = np.array([int(sbits, 16)], np.uint32).view(np.float32)[0]
        ref = (np.float32(1.0) / sc).view(np.uint32)
        assert int(rbits, 16) == int(ref), (b, sbits, rbits, hex(int(ref)))
        # and the decode itself is decode_e4m3 (fp4.py:59-66)
        e, m = int(b) >> 3, int(b) & 7
        want = m * 2.0 ** -9 if e == 0 else (1 + m / 8) * 2.0 ** (e - 7)
        assert float(sc) == want
