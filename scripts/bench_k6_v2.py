"""K6 down GEMM on the Kimi EP8 hot rank (8 experts x ~17.1 k rows, N = 2048,
K = 1408): v1 (1-CTA 128x256) vs v2 (gemm_fp4_pair.cu: 2-SM pairs, A resident,
N = 128 double-buffered) vs one dense cuBLASLt NVFP4 GEMM of the same flops;
interleaved, NVML clocks. v2 with REALB_DBG_FP4=1 (no stores) beside it."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "scripts")]
import numpy as np, torch
from bench_fp4 import interleaved
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.quant import quantize_nvfp4

os.environ.pop("REALB_GEMM_CLUSTER", None)
E = 8
counts = ((np.random.default_rng(0).random(E) * 0.2 + 0.9) * 17134).astype(np.int64)
M = int(counts.sum())
lay, rows = host_layout(counts, np.ones(E, np.int64))
lt = torch.from_numpy(lay).cuda()
sp = _lib.stream_ptr()
shapes = [("gate_up", 2816, 2048), ("down", 2048, 1408)]
out = {"rows": M}
with ClockSampler(0) as clk:
    for name, N, K in shapes:
        A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
        ac, asf = quantize_nvfp4(A)
        wc, wsf = quantize_nvfp4(W)
        o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
        hc = torch.empty(rows, N // 4, dtype=torch.uint8, device="cuda")
        hs = torch.empty(rows * (N // 2) // 16, dtype=torch.uint8, device="cuda")
        epi = _lib.EPI_SWIGLU if name == "gate_up" else _lib.EPI_STORE
        f = (lambda ac=ac, asf=asf, wc=wc, wsf=wsf, N=N, K=K, o=o, hc=hc, hs=hs, epi=epi: _lib.call(
            "realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(), rows, N, K, E,
            lt.data_ptr(), epi, None if epi == _lib.EPI_SWIGLU else o.data_ptr(), hc.data_ptr(), hs.data_ptr(), 0,
            sp))
        variants = {f"{name}_v1": ({"REALB_K6_VERSION": "1", "REALB_DBG_FP4": "0"}, f),
                    f"{name}_v1_pair": ({"REALB_K6_VERSION": "1", "REALB_DBG_FP4": "0", "REALB_GEMM_CLUSTER": "2"}, f),
                    f"{name}_v2": ({"REALB_K6_VERSION": "2", "REALB_DBG_FP4": "0"}, f),
                    f"{name}_v2_nostore": ({"REALB_K6_VERSION": "2", "REALB_DBG_FP4": "1"}, f)}
        for d in os.environ.get("K6_VDBG", "").split(",") if os.environ.get("K6_VDBG") else []:
            for r in os.environ.get("K6_VDBG_RUN", "").split(","):
                variants[f"{name}_v2_dbg{d}_run{r}"] = ({"REALB_K6_VERSION": "2", "REALB_DBG_FP4": d,
                                                         "REALB_K6_RUN": r}, f)
        for r in os.environ.get("K6_RUN", "").split(",") if os.environ.get("K6_RUN") else []:
            variants[f"{name}_v2_run{r}"] = ({"REALB_K6_VERSION": "2", "REALB_DBG_FP4": "0", "REALB_K6_RUN": r}, f)
        for w in os.environ.get("K6_WAIT", "0").split(","):
            for d in [0] + list(map(int, os.environ.get("K6_DBG", "").split(",") if os.environ.get("K6_DBG") else [])):
                if w == "0" and d == 0:
                    continue
                variants[f"{name}_v2_w{w}_dbg{d}"] = ({"REALB_K6_VERSION": "2", "REALB_DBG_FP4": str(d),
                                                       "REALB_DBG_WAIT": w}, f)
        for v in variants.values():
            v[0].setdefault("REALB_K6_RUN", "")
            v[0].setdefault("REALB_GEMM_CLUSTER", "")
        a = torch.randint(0, 255, (M, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 255, (N, K // 2), dtype=torch.uint8, device="cuda").view(torch.float4_e2m1fn_x2)
        Mp = (M + 127) // 128 * 128
        sa = torch.full((Mp * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
        sb = torch.full((N * K // 16,), 1.0, device="cuda").to(torch.float8_e4m3fn)
        variants[f"{name}_cublaslt_dense"] = ({}, lambda a=a, b=b, sa=sa, sb=sb: torch._scaled_mm(
            a, b.t(), sa, sb, out_dtype=torch.bfloat16))
        res = interleaved(variants, rounds=6, per=8)
        flops = 2.0 * M * N * K
        for k, ms in res.items():
            out[k] = {"ms": ms, "pflops": flops / ms / 1e12}
        print(name, {k: round(v, 4) for k, v in res.items()}, flush=True)
os.environ["REALB_DBG_FP4"] = "0"
os.environ.pop("REALB_K6_VERSION", None)
out["clocks"] = clk.summary()
print(json.dumps(out, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "bench_k6_v2.json"), "w"), indent=1)
