"""One ncu-capturable launch of a K6 variant on the Kimi EP8 hot-rank shape
(8 experts x ~17.1 k rows), between cudaProfilerStart/Stop (run ncu with
--profile-from-start off). argv: which in {k6_down, k6_gate_up, cublaslt_down,
cublaslt_gate_up}; REALB_GEMM_CLUSTER etc. from the environment."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.quant import quantize_nvfp4

which = sys.argv[1]
E = 8
counts = ((np.random.default_rng(0).random(E) * 0.2 + 0.9) * 17134).astype(np.int64)
M = int(counts.sum())
lay, rows = host_layout(counts, np.ones(E, np.int64))
lt = torch.from_numpy(lay).cuda()
sp = _lib.stream_ptr()
N, K = (2816, 2048) if which.endswith("gate_up") else (2048, 1408)
if which.startswith("k6"):
    A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
    ac, asf = quantize_nvfp4(A)
    wc, wsf = quantize_nvfp4(W)
    o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    hc = torch.empty(rows, N // 4, dtype=torch.uint8, device="cuda")
    hs = torch.empty(rows * (N // 2) // 16, dtype=torch.uint8, device="cuda")
    epi = _lib.EPI_SWIGLU if which.endswith("gate_up") else _lib.EPI_STORE
    f = lambda: _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
                          rows, N, K, E, lt.data_ptr(), epi, None if epi == _lib.EPI_SWIGLU else o.data_ptr(),
                          hc.data_ptr(), hs.data_ptr(), 0, sp)
else:
    a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    Mp = (M + 127) // 128 * 128
    sa = torch.full((Mp * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    sb = torch.full((N * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
for _ in range(5):
    f()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
f()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", which, rows)
