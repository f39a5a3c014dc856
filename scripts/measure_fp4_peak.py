"""Measured dense NVFP4 peak of this B200 (the roofline denominator for K6):
cuBLASLt block-scaled NVFP4 GEMM (torch._scaled_mm, E2M1 x E2M1 with UE4M3
1x16 block scales, bf16 out), M = N = K = 8192 (2 N^3 flops), timed the way
MEASURED_PEAKS.json times bf16: best of 10 single launches with CUDA events
(burst) and back to back for 4 s (sustained), NVML clocks sampled during both.
Also the bf16 cuBLAS figure on the same box for reference.

  python scripts/measure_fp4_peak.py  -> profiles/r02/fp4_peak.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2604_19503_b200.clocks import ClockSampler  # noqa: E402

N = 8192


def fp4_operands(n):
    a = torch.randint(0, 255, (n, n // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 255, (n, n // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
    sa = torch.full((n * n // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    sb = torch.full((n * n // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
    return lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)


def bf16_operands(n):
    a = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    b = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    return lambda: torch.matmul(a, b)


def burst(fn, reps=10):
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        time.sleep(0.02)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best / 1e3


def sustained(fn, seconds=4.0):
    fn()
    torch.cuda.synchronize()
    n = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / 1e3 / n


def main():
    flops = 2.0 * N ** 3
    out = {"shape": f"{N}^3", "flops": flops, "gpu": torch.cuda.get_device_name(0)}
    for name, mk in (("nvfp4", fp4_operands), ("bf16", bf16_operands)):
        fn = mk(N)
        for _ in range(3):
            fn()
        with ClockSampler(0) as ck:
            tb = burst(fn)
        with ClockSampler(0) as cs:
            ts = sustained(fn)
        out[name] = {"burst_tflops": flops / tb / 1e12, "burst_ms": tb * 1e3, "burst_clocks": ck.summary(),
                     "sustained_tflops": flops / ts / 1e12, "sustained_ms": ts * 1e3, "sustained_clocks": cs.summary()}
        del fn
        torch.cuda.empty_cache()
    out["how"] = ("torch._scaled_mm NVFP4 (cuBLASLt, 1x16 UE4M3 block scales, bf16 out) and torch.matmul bf16, "
                  f"{N}^3: best of 10 launches after 20 ms idle (burst) and back to back for 4 s (sustained)")
    os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "fp4_peak.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
