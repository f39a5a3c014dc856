"""Is the grouped gate_up GEMM bound by the chip (clock / power) or by its own
tiling? Times, interleaved with NVML clocks: K5 gate_up on the 1-GPU Kimi layer
(64 experts x ~768 rows), torch._grouped_mm on the same rows, and cuBLAS dense
bf16 GEMMs of the same total flops ([49152 x 2048] @ [2048 x 2816]) and of the
8192^3 peak shape."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from bench_fp4 import interleaved

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
P = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
offs = torch.tensor(np.cumsum((counts + 127) // 128 * 128), dtype=torch.int32, device="cuda")
Wt = W.view(E, N, K).transpose(1, 2)
sp = _lib.stream_ptr()
variants = {
    "k5_gate_up": ({}, lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E,
                                         lt.data_ptr(), 0, _lib.EPI_SWIGLU, o.data_ptr(), 0, sp)),
    "torch_grouped_mm": ({}, lambda: torch._grouped_mm(A, Wt, offs=offs)),
    "cublas_dense_same_flops": ({}, lambda: Ad @ Wd),
    "cublas_8192cube": ({}, lambda: P @ P),
}
with ClockSampler(0) as clk:
    res = interleaved(variants, rounds=8, per=10)
fl = {"k5_gate_up": 2.0 * M * N * K, "torch_grouped_mm": 2.0 * M * N * K, "cublas_dense_same_flops": 2.0 * M * N * K,
      "cublas_8192cube": 2.0 * 8192**3}
out = {k: {"ms": v, "tflops": fl[k] / v / 1e9} for k, v in res.items()}
out["clocks"] = clk.summary()
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_dense_ref.json", "w"), indent=1)
