"""K6 on the EP8 hot rank: how much of each GEMM is the single-accumulator
hand-off between tiles (REALB_DBG_FP4 bits, interleaved): full; 1 = drain, no
stores; 8 = released unread; 16 = no hand-off at all (mainloop alone, wrong
results); STORE only: 32 = staged but not stored, 64 = every store to tile 0
(no HBM write-back). 1-CTA and 2-CTA pair forms."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "scripts")]
import numpy as np, torch
from bench_fp4 import interleaved
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.quant import quantize_nvfp4

E = 8
counts = ((np.random.default_rng(0).random(E) * 0.2 + 0.9) * 17134).astype(np.int64)
lay, rows = host_layout(counts, np.ones(E, np.int64))
lt = torch.from_numpy(lay).cuda()
sp = _lib.stream_ptr()
out = {"rows": int(counts.sum())}
with ClockSampler(0) as clk:
    for name, N, K, epi in (("gate_up", 2816, 2048, _lib.EPI_SWIGLU), ("down", 2048, 1408, _lib.EPI_STORE)):
        A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
        ac, asf = quantize_nvfp4(A)
        wc, wsf = quantize_nvfp4(W)
        o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
        hc = torch.empty(rows, N // 4, dtype=torch.uint8, device="cuda")
        hs = torch.empty(rows * (N // 2) // 16, dtype=torch.uint8, device="cuda")
        f = (lambda ac=ac, asf=asf, wc=wc, wsf=wsf, N=N, K=K, o=o, hc=hc, hs=hs, epi=epi: _lib.call(
            "realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(), rows, N, K, E,
            lt.data_ptr(), epi, None if epi == _lib.EPI_SWIGLU else o.data_ptr(), hc.data_ptr(), hs.data_ptr(), 0, sp))
        dbgs = (0, 1, 8, 16) + ((32, 64) if epi == _lib.EPI_STORE else ())
        variants = {f"{name}_cl{cl}_dbg{d}": ({"REALB_GEMM_CLUSTER": cl, "REALB_DBG_FP4": str(d)}, f)
                    for cl in ("1", "2") for d in dbgs}
        res = interleaved(variants, rounds=5, per=6)
        flops = 2.0 * counts.sum() * N * K
        for k, ms in res.items():
            out[k] = {"ms": ms, "pflops": flops / ms / 1e12}
        print(name, {k: round(v, 4) for k, v in res.items()}, flush=True)
os.environ["REALB_DBG_FP4"] = "0"
os.environ.pop("REALB_GEMM_CLUSTER", None)
out["clocks"] = clk.summary()
print(json.dumps(out, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "bench_k6_bubble.json"), "w"), indent=1)
