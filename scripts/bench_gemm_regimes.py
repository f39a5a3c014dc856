"""K5 1-CTA vs 2-CTA pair vs cuBLAS dense (same flops) on the 1-GPU Kimi gate_up,
in two regimes: "sustained" (each variant launched back to back, interleaved
rounds: the power-capped steady state a long layer step sees) and "burst"
(single launches separated by idle gaps: clocks near maximum, as the bench's
roofline timing sees them). NVML clocks per regime."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from bench_fp4 import interleaved, ev_time

E, N, K, per = 64, 2816, 2048, 768
rng = np.random.default_rng(0)
counts = ((rng.random(E) * 0.4 + 0.8) * per).astype(np.int64)
lay, rows = host_layout(counts, np.zeros(E, np.int64))
A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
W = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
lt = torch.from_numpy(lay).cuda()
o = torch.empty(rows, N // 2, dtype=torch.bfloat16, device="cuda")
M = int(counts.sum())
Ad = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Wd = (torch.randn(K, N, device="cuda") / K**0.5).to(torch.bfloat16)
sp = _lib.stream_ptr()
k5 = lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E, lt.data_ptr(), 0,
                       _lib.EPI_SWIGLU, o.data_ptr(), 0, sp)
variants = {"k5_cta1": ({"REALB_GEMM_CLUSTER": "1"}, k5), "k5_pair": ({"REALB_GEMM_CLUSTER": "2"}, k5),
            "cublas_dense": ({}, lambda: Ad @ Wd)}
out = {"flops": 2.0 * M * N * K}
with ClockSampler(0) as clk:
    out["sustained_ms"] = interleaved(variants, rounds=8, per=10)
out["sustained_clocks"] = clk.summary()
with ClockSampler(0) as clk:
    samples = {k: [] for k in variants}
    for _ in range(12):
        for name, (env, fn) in variants.items():
            os.environ.update(env)
            torch.cuda.synchronize()
            time.sleep(0.02)  # idle gap: clocks recover
            samples[name].append(ev_time(fn))
    out["burst_ms"] = {k: float(np.median(v)) for k, v in samples.items()}
out["burst_clocks"] = clk.summary()
os.environ["REALB_GEMM_CLUSTER"] = "1"
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_gemm_regimes.json", "w"), indent=1)
