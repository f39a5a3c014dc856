"""Router microbenchmark with debug variants (REALB_DBG_ROUTER: 1 no epilogue, 4 no loads,
16 no logits stores, 32 in-kernel phase cycles written into topk_w; REALB_ROUTER_STAGES caps
the ring depth). BENCH_T / BENCH_STAGES / BENCH_DBG select the runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch
shape = SHAPES["kimi"]
for T in [int(t) for t in os.environ.get("BENCH_T", "8192,65536").split(",")]:
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T))
    E, k, H = 64, 6, 2048
    logits = torch.empty(T, E, device="cuda"); idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    w = torch.empty(T, k, device="cuda"); cc = torch.empty((T + 63) // 64, E, 2, dtype=torch.int32, device="cuda")
    bias = torch.zeros(E, device="cuda")
    f = lambda: _lib.call("realb_router_topk_stats", x.data_ptr(), router.data_ptr(), bias.data_ptr(), mod.data_ptr(), T, H, E, k, 1, 2.446, 1e-12, logits.data_ptr(), idx.data_ptr(), w.data_ptr(), cc.data_ptr(), _lib.stream_ptr())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    for stages, dbg in [(s_, d_) for s_ in os.environ.get("BENCH_STAGES", "12").split(",")
                        for d_ in os.environ.get("BENCH_DBG", "0,1,4,5").split(",")]:
        os.environ["REALB_ROUTER_STAGES"] = stages
        if True:
            os.environ["REALB_DBG_ROUTER"] = str(dbg)
            for _ in range(3): f()
            torch.cuda.synchronize()
            ts = []
            for _ in range(15):
                flush.zero_()  # x comes from HBM, as inside the layer step
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                a.record(); f(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
            t = sorted(ts)[7]
            if dbg == "32":
                st = w.view(torch.int32)[::64, :6].cpu()
                print("phase cycles (done, pass1+b1, merge+b2, pass2+b3, select, out+bar): median",
                      st.median(dim=0).values.tolist(), "max", st.max(dim=0).values.tolist())
            print(f"T={T} stages={stages} dbg={dbg} {t*1e3:8.1f} us  {T*H*2/t/1e6:8.1f} GB/s (x only, event-timed)", flush=True)
