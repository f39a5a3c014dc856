"""Microbenchmark: grouped NVFP4 tcgen05 GEMM on the Kimi EP8 hot-rank shape —
1-CTA vs 2-CTA-pair kernels and debug variants (REALB_DBG_FP4: 1 = no epilogue
math/stores, 2 = no scale copies, 4 = no MMAs), next to the BF16 kernel on the same
rows and cuBLASLt dense NVFP4 (torch._scaled_mm) as a measured FP4 reference peak.

Variants are timed interleaved (round-robin, several rounds, median of each
variant's samples) so clock / power drift hits every variant alike; NVML SM
clocks are sampled throughout."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.quant import quantize_nvfp4


def ev_time(fn):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); fn(); b.record(); b.synchronize()
    return a.elapsed_time(b)


def interleaved(variants, rounds=6, per=8):
    """variants: {name: (env dict, fn)} -> {name: median ms}"""
    samples = {k: [] for k in variants}
    for name, (env, fn) in variants.items():  # warm every variant
        os.environ.update(env)
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    for _ in range(rounds):
        for name, (env, fn) in variants.items():
            os.environ.update(env)
            for _ in range(per):
                samples[name].append(ev_time(fn))
    return {k: float(np.median(v)) for k, v in samples.items()}


def main():
    out = {}
    E = 8
    counts = np.full(E, 17134, np.int64)   # Kimi EP8 hot rank: 137K pairs over 8 experts
    dbgs = [int(d) for d in os.environ.get("BENCH_DBG", "0,1,7").split(",")]
    with ClockSampler(0) as clk:
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
            f = lambda: _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(),
                                  wsf.data_ptr(), rows, N, K, E, lt.data_ptr(), epi, o.data_ptr(), hc.data_ptr(),
                                  hsf.data_ptr(), 0, _lib.stream_ptr())
            lay0, _ = host_layout(counts, np.zeros(E, np.int64))
            lt0 = torch.from_numpy(lay0).cuda()
            g = lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E,
                                  lt0.data_ptr(), 0, epi, o.data_ptr(), 0, _lib.stream_ptr())
            variants = {f"fp4_{label}_cl{cl}_dbg{d}": ({"REALB_GEMM_CLUSTER": cl, "REALB_DBG_FP4": str(d)}, f)
                        for cl in ("1", "2") for d in dbgs}
            variants[f"bf16_{label}"] = ({"REALB_GEMM_CLUSTER": "2", "REALB_DBG_FP4": "0"}, g)
            res = interleaved(variants)
            for k, ms in res.items():
                out[k] = dict(ms=ms, tflops=flops / ms / 1e9)
            print(label, {k: round(v, 4) for k, v in res.items()}, flush=True)
        os.environ.pop("REALB_GEMM_CLUSTER", None)
        os.environ["REALB_DBG_FP4"] = "0"
        # cuBLASLt dense NVFP4 / BF16 (measured reference peaks)
        try:
            M = N = K = 8192
            a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
            b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
            sa = torch.full((M * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
            sb = torch.full((N * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
            x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            y = torch.randn(N, K, device="cuda").to(torch.bfloat16)
            res = interleaved({
                "cublas_nvfp4_dense_8192": ({}, lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)),
                "cublas_bf16_dense_8192": ({}, lambda: x @ y.t())}, rounds=3)
            for k, ms in res.items():
                out[k] = dict(ms=ms, tflops=2.0 * M * N * K / ms / 1e9)
        except Exception as e:
            out["cublas_dense_8192"] = repr(e)[:300]
    out["clocks"] = clk.summary()
    print(json.dumps(out, indent=1))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/bench_fp4.json", "w"), indent=1)


if __name__ == "__main__":
    main()
