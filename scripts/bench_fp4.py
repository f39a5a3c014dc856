"""Microbenchmark: grouped NVFP4 tcgen05 GEMM on the Kimi EP8 hot-rank shape, with
debug variants (REALB_DBG_FP4: 1 = no epilogue math, 2 = no scale copies), next to the
BF16 kernel on the same rows and cuBLASLt dense NVFP4 (torch._scaled_mm) as a
measured FP4 reference peak."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.quant import quantize_nvfp4

def timeit(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(it):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]

out = {}
E = 8
counts = np.full(E, 17134, np.int64)   # Kimi EP8 hot rank: 137K pairs over 8 experts
for label, N, K, epi in [("gate_up", 2816, 2048, _lib.EPI_SWIGLU), ("down", 2048, 1408, _lib.EPI_STORE)]:
    lay, rows = host_layout(counts, np.ones(E, np.int64))
    lt = torch.from_numpy(lay).cuda()
    A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
    ac, asf = quantize_nvfp4(A); wc, wsf = quantize_nvfp4(W)
    o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    hc = torch.empty(rows, N // 4, dtype=torch.uint8, device="cuda")
    hsf = torch.empty(rows * N // 32, dtype=torch.uint8, device="cuda")
    flops = 2.0 * counts.sum() * N * K
    for dbg in (0, 1, 2, 3, 7, 8, 16, 24):
        os.environ["REALB_DBG_FP4"] = str(dbg)
        f = lambda: _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
                              rows, N, K, E, lt.data_ptr(), epi, o.data_ptr(), hc.data_ptr(), hsf.data_ptr(), 0, _lib.stream_ptr())
        t = timeit(f)
        out[f"fp4_{label}_dbg{dbg}"] = dict(ms=t, tflops=flops / t / 1e9)
    os.environ["REALB_DBG_FP4"] = "0"
    lay0, _ = host_layout(counts, np.zeros(E, np.int64))
    lt0 = torch.from_numpy(lay0).cuda()
    g = lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E, lt0.data_ptr(), 0, epi,
                          o.data_ptr(), 0, _lib.stream_ptr())
    t = timeit(g)
    out[f"bf16_{label}"] = dict(ms=t, tflops=flops / t / 1e9)
    print(label, {k: v for k, v in out.items() if label in k}, flush=True)

# cuBLASLt dense NVFP4 (measured FP4 reference peak)
try:
    M = N = K = 8192
    a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    sa = torch.full((M * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    sb = torch.full((N * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    h = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
    t = timeit(h)
    out["cublas_nvfp4_dense_8192"] = dict(ms=t, tflops=2.0 * M * N * K / t / 1e9)
except Exception as e:
    out["cublas_nvfp4_dense_8192"] = repr(e)[:300]
try:
    M = N = K = 8192
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    t = timeit(lambda: a @ b.t())
    out["cublas_bf16_dense_8192"] = dict(ms=t, tflops=2.0 * M * N * K / t / 1e9)
except Exception as e:
    out["cublas_bf16_dense_8192"] = repr(e)[:200]
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_fp4.json", "w"), indent=1)
