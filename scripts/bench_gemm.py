"""Microbenchmark: grouped BF16 tcgen05 GEMM (1-CTA and 2-CTA-pair forms, STORE and
SwiGLU epilogues, debug variants REALB_DBG_BF16 1 = no epilogue, 4 = no MMA,
5 = TMA only) vs torch._grouped_mm on the Kimi / Qwen shapes, timed interleaved
(round-robin over variants, median per variant) with NVML clocks sampled."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from bench_fp4 import interleaved

SHAPES = [("kimi_gate_up_1gpu", 64, 2816, 2048, 768), ("kimi_down_1gpu", 64, 2048, 1408, 768),
          ("kimi_gate_up_ep8hot", 8, 2816, 2048, 13000), ("qwen_gate_up_1gpu", 128, 1536, 2048, 512)]


def main():
    out = {}
    rng = np.random.default_rng(0)
    only = os.environ.get("BENCH_SHAPES")
    dbgs = [int(d) for d in os.environ.get("BENCH_DBG", "0").split(",")]
    with ClockSampler(0) as clk:
        for label, E, N, K, per in SHAPES:
            if only and label not in only.split(","):
                continue
            counts = ((rng.random(E) * 0.4 + 0.8) * per).astype(np.int64)
            if os.environ.get("BENCH_EVEN"):  # whole 256-row units: no 2-SM pair dummy m-tiles
                counts = np.maximum(256, (counts + 128) // 256 * 256)
            lay, rows = host_layout(counts, np.zeros(E, np.int64))
            A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
            W = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
            lt = torch.from_numpy(lay).cuda()
            o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
            epi = _lib.EPI_SWIGLU if "gate_up" in label else _lib.EPI_STORE
            f = lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E, lt.data_ptr(),
                                  0, epi, o.data_ptr(), 0, _lib.stream_ptr())
            orders = os.environ.get("BENCH_ORDER", "m").split(",")
            variants = {f"cl{cl}_dbg{d}_{o}": ({"REALB_GEMM_CLUSTER": cl, "REALB_DBG_BF16": str(d),
                                                "REALB_GEMM_ORDER": o}, f)
                        for cl in os.environ.get("BENCH_CL", "1,2").split(",") for d in dbgs for o in orders}
            offs = torch.tensor(np.cumsum((counts + 127) // 128 * 128), dtype=torch.int32, device="cuda")
            Wt = W.view(E, N, K).transpose(1, 2)
            variants["torch_grouped_mm"] = ({}, lambda: torch._grouped_mm(A, Wt, offs=offs))
            res = interleaved(variants)
            valid = 2.0 * counts.sum() * N * K
            out[label] = {k: dict(ms=ms, valid_tflops=valid / ms / 1e9) for k, ms in res.items()}
            print(label, {k: round(v, 4) for k, v in res.items()}, flush=True)
    os.environ["REALB_DBG_BF16"] = "0"
    os.environ.pop("REALB_GEMM_CLUSTER", None)
    out["clocks"] = clk.summary()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/bench_gemm.json", "w"), indent=1)


if __name__ == "__main__":
    main()
