"""Microbenchmark: grouped BF16 tcgen05 GEMM vs torch._grouped_mm on Kimi EP-rank shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from helpers import host_layout
from paper_2604_19503_b200 import _lib

def timeit(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(it):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts)//2]

out = {}
rng = np.random.default_rng(0)
for label, E, N, K, per in [("kimi_gate_up_ep8hot", 8, 2816, 2048, 13000), ("kimi_down_ep8hot", 8, 2048, 1408, 13000),
                            ("kimi_gate_up_1gpu", 64, 2816, 2048, 768), ("qwen_gate_up_1gpu", 128, 1536, 2048, 512),
                            ("square", 1, 4096, 4096, 8192)]:
    counts = (rng.random(E) * 0.4 + 0.8) * per
    counts = counts.astype(np.int64)
    lay, rows = host_layout(counts, np.zeros(E, np.int64))
    A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
    lt = torch.from_numpy(lay).cuda()
    o = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    f = lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E, lt.data_ptr(), 0, 0, o.data_ptr(), 0, _lib.stream_ptr())
    t = timeit(f)
    flops = 2.0 * rows * N * K
    dbgt = {}
    for dbg in (1, 4, 5):
        os.environ["REALB_DBG_BF16"] = str(dbg)
        dbgt[dbg] = timeit(f)
    os.environ["REALB_DBG_BF16"] = "0"
    fs = lambda: _lib.call("realb_grouped_gemm_bf16", A.data_ptr(), W.data_ptr(), rows, N, K, E, lt.data_ptr(), 0, 1, o.data_ptr(), 0, _lib.stream_ptr())
    t_swiglu = timeit(fs)
    # torch grouped mm on the same padded rows
    offs = torch.tensor(np.cumsum((counts + 127)//128*128), dtype=torch.int32, device="cuda")
    Wt = W.view(E, N, K).transpose(1, 2)
    g = lambda: torch._grouped_mm(A, Wt, offs=offs)
    try:
        tg = timeit(g)
    except Exception as e:
        tg = repr(e)[:100]
    cl = {}
    for c in ("1", "2"):
        os.environ["REALB_GEMM_CLUSTER"] = c
        cl[c] = (timeit(f), timeit(fs))
    del os.environ["REALB_GEMM_CLUSTER"]
    valid = 2.0 * counts.sum() * N * K
    out[label] = dict(rows=rows, ms=t, tflops=flops / t / 1e9, valid_tflops=valid / t / 1e9,
                      cluster_ms={c: v for c, v in cl.items()},
                      cluster_valid_tflops={c: (valid / v[0] / 1e9, valid / v[1] / 1e9) for c, v in cl.items()},
                      ms_swiglu=t_swiglu, ms_no_epi=dbgt[1],
                      ms_no_mma=dbgt[4], ms_tma_only=dbgt[5], torch_ms=tg,
                      torch_tflops=(flops / tg / 1e9) if isinstance(tg, float) else None)
    print(label, out[label], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_gemm.json", "w"), indent=1)
