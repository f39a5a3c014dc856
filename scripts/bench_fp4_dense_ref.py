"""K6 (grouped NVFP4) on the Kimi EP8 hot rank (8 experts x ~17.1 k rows) vs ONE
cuBLASLt dense NVFP4 GEMM of the same flops (torch._scaled_mm, bf16 out), for the
gate_up (N = 2816, K = 2048) and down (N = 2048, K = 1408) shapes; interleaved,
NVML clocks. K6 gate_up also runs its SwiGLU + NVFP4 re-quantisation epilogue."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "scripts")]
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.quant import quantize_nvfp4
from bench_fp4 import interleaved

E = 8
rng = np.random.default_rng(0)
counts = ((rng.random(E) * 0.2 + 0.9) * 17134).astype(np.int64)
M = int(counts.sum())
lay, rows = host_layout(counts, np.ones(E, np.int64))
lt = torch.from_numpy(lay).cuda()
sp = _lib.stream_ptr()
out = {"rows": M}
variants, flops = {}, {}
for name, N, K, epi in (("gate_up", 2816, 2048, _lib.EPI_SWIGLU), ("down", 2048, 1408, _lib.EPI_STORE)):
    A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
    ac, asf = quantize_nvfp4(A)
    wc, wsf = quantize_nvfp4(W)
    o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    hc = torch.empty(rows, N // 4, dtype=torch.uint8, device="cuda")
    hs = torch.empty(rows * (N // 2) // 16, dtype=torch.uint8, device="cuda")
    if epi == _lib.EPI_SWIGLU:
        f = (lambda ac=ac, asf=asf, wc=wc, wsf=wsf, N=N, K=K, hc=hc, hs=hs: _lib.call(
            "realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(), rows, N, K, E,
            lt.data_ptr(), _lib.EPI_SWIGLU, None, hc.data_ptr(), hs.data_ptr(), 0, sp))
    else:
        f = (lambda ac=ac, asf=asf, wc=wc, wsf=wsf, N=N, K=K, o=o: _lib.call(
            "realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(), rows, N, K, E,
            lt.data_ptr(), _lib.EPI_STORE, o.data_ptr(), None, None, 0, sp))
    variants[f"k6_{name}"] = ({}, f)
    flops[f"k6_{name}"] = 2.0 * M * N * K
    a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    Mp = (M + 127) // 128 * 128
    sa = torch.full((Mp * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    sb = torch.full((N * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    try:
        torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
        variants[f"cublaslt_dense_{name}"] = ({}, lambda a=a, b=b, sa=sa, sb=sb: torch._scaled_mm(
            a, b.t(), sa, sb, out_dtype=torch.bfloat16))
        flops[f"cublaslt_dense_{name}"] = 2.0 * M * N * K
    except Exception as e:
        out[f"cublaslt_dense_{name}"] = repr(e)[:300]
with ClockSampler(0) as clk:
    res = interleaved(variants, rounds=6, per=8)
for k, ms in res.items():
    out[k] = {"ms": ms, "pflops": flops[k] / ms / 1e12}
out["clocks"] = clk.summary()
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_fp4_dense_ref.json", "w"), indent=1)
