"""K6 down GEMM (EP8 hot rank: 8 experts x ~17.1 k rows, N = 2048, K = 1408): how much
of it is the operand feed of the 3-stage ring the STORE epilogue's 48 KB staging
leaves room for. Interleaved variants:
  full           the shipped kernel (3 stages, TMA-store epilogue)
  nostore_3st    REALB_DBG_FP4=1: accumulator drained, no convert / stores (3 stages)
  nostore_4st    the same with 4 operand stages (REALB_DBG_FP4_STORE4=1, experiment only)
  release_3st    REALB_DBG_FP4=9: accumulator released unread"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "scripts")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench_fp4 import interleaved  # noqa: E402
from helpers import host_layout  # noqa: E402
from paper_2604_19503_b200 import _lib  # noqa: E402
from paper_2604_19503_b200.clocks import ClockSampler  # noqa: E402
from paper_2604_19503_b200.quant import quantize_nvfp4  # noqa: E402

E, N, K = 8, 2048, 1408
counts = ((np.random.default_rng(0).random(E) * 0.2 + 0.9) * 17134).astype(np.int64)
lay, rows = host_layout(counts, np.ones(E, np.int64))
lt = torch.from_numpy(lay).cuda()
A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
ac, asf = quantize_nvfp4(A)
wc, wsf = quantize_nvfp4(W)
o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
f = lambda: _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(), rows,
                      N, K, E, lt.data_ptr(), _lib.EPI_STORE, o.data_ptr(), None, None, 0, _lib.stream_ptr())
base = {"REALB_DBG_FP4_STORE4": "0"}
variants = {"full": (dict(base, REALB_DBG_FP4="0"), f),
            "nostore_3st": (dict(base, REALB_DBG_FP4="1"), f),
            "nostore_4st": ({"REALB_DBG_FP4": "1", "REALB_DBG_FP4_STORE4": "1"}, f),
            "release_3st": (dict(base, REALB_DBG_FP4="9"), f)}
with ClockSampler(0) as clk:
    res = interleaved(variants, rounds=6, per=8)
os.environ.update({"REALB_DBG_FP4": "0", "REALB_DBG_FP4_STORE4": "0"})
flops = 2.0 * counts.sum() * N * K
out = {k: {"ms": v, "pflops": flops / v / 1e12} for k, v in res.items()}
out["clocks"] = clk.summary()
out["rows"] = int(counts.sum())
print(json.dumps(out, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "bench_k6_stages.json"), "w"), indent=1)
