"""Microbenchmark: the EP hot rank's down GEMM followed by the return copy
(STORE into a local buffer + realb_index_rows into the return layout, the
unfused path) vs the fused scatter epilogue (realb_grouped_gemm_*_scatter,
rows stored straight to their per-source destination), for the BF16 and the
NVFP4 down GEMM at the Kimi EP8 hot-rank shape (8 experts x ~17.1 k rows,
N = H = 2048, K = I = 1408). One GPU: the 8 destinations are local buffers, so
this measures the epilogue cost, not NVLink. Interleaved timing, NVML clocks.

  python scripts/bench_scatter.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    import numpy as np
    import torch

    from bench_fp4 import interleaved
    from helpers import host_layout
    from paper_2604_19503_b200 import _lib
    from paper_2604_19503_b200.clocks import ClockSampler
    from paper_2604_19503_b200.quant import quantize_nvfp4

    torch.cuda.set_device(0)
    E, N, K, R = 8, 2048, 1408, 8
    rng = np.random.default_rng(0)
    counts = ((rng.random(E) * 0.2 + 0.9) * 17134).astype(np.int64)
    out = {}
    for prec in (0, 1):
        lay, rows = host_layout(counts, np.full(E, prec, np.int64))
        lay_t = torch.from_numpy(lay).cuda()
        A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(E * N, K, device="cuda") * 0.02).to(torch.bfloat16)
        valid = np.concatenate([int(lay[8 + e]) + np.arange(c) for e, c in enumerate(counts)])
        d = rng.integers(0, R, len(valid))
        m = np.full(rows, -1, np.int32)
        sizes = []
        for dd in range(R):
            sel = valid[d == dd]
            m[sel] = (dd << 25) | np.arange(len(sel))
            sizes.append(len(sel))
        m_t = torch.from_numpy(m).cuda()
        dsts = [torch.empty(s + 1, N, dtype=torch.bfloat16, device="cuda") for s in sizes]
        bases = np.array([t.data_ptr() for t in dsts], np.uint64)
        # unfused: STORE, then a row copy into one return buffer in (destination, row) order
        order = np.argsort(m[valid], kind="stable")
        idx_t = torch.from_numpy(valid[order].astype(np.int32)).cuda()
        rows_out = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
        ret = torch.empty(len(valid), N, dtype=torch.bfloat16, device="cuda")
        sp = _lib.stream_ptr()
        if prec == 0:
            def store():
                _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E, lay_t.data_ptr(),
                          0, _lib.EPI_STORE, rows_out.data_ptr(), 0, sp)

            def scatter():
                _lib.call("realb_grouped_gemm_bf16_scatter", A.data_ptr(), W.data_ptr(), rows, N, K, E,
                          lay_t.data_ptr(), 0, m_t.data_ptr(), R, bases.ctypes.data, 0, sp)
        else:
            ac, asf = quantize_nvfp4(A)
            wc, wsf = quantize_nvfp4(W)

            def store():
                _lib.call("realb_grouped_gemm_nvfp4", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(), wsf.data_ptr(),
                          rows, N, K, E, lay_t.data_ptr(), _lib.EPI_STORE, rows_out.data_ptr(), None, None, 0, sp)

            def scatter():
                _lib.call("realb_grouped_gemm_nvfp4_scatter", ac.data_ptr(), asf.data_ptr(), wc.data_ptr(),
                          wsf.data_ptr(), rows, N, K, E, lay_t.data_ptr(), m_t.data_ptr(), R, bases.ctypes.data,
                          0, sp)

        def copy():
            _lib.call("realb_index_rows", rows_out.data_ptr(), idx_t.data_ptr(), len(valid), N, ret.data_ptr(), sp)

        def unfused():
            store()
            copy()

        with ClockSampler(0) as clk:
            res = interleaved({"store": ({}, store), "copy": ({}, copy), "store+copy": ({}, unfused),
                               "scatter": ({}, scatter)})
        name = "bf16" if prec == 0 else "nvfp4"
        out[name] = {"ms": res, "rows": int(len(valid)), "clocks": clk.summary()}
        print(name, json.dumps(out[name]), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/bench_scatter.json", "w"), indent=1)


if __name__ == "__main__":
    main()
