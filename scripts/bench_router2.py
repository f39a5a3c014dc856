"""Router fixed-cost probe: tiny (T, H) cases next to a 64-element torch fill_ timed the
same way (CUDA events around one launch), which gives the launch / event overhead."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_19503_b200 import _lib
E, k = 64, 6
for T in (64, 8192):
    for H in (64, 512, 2048):
        x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
        router = torch.randn(E, H, device="cuda").to(torch.bfloat16)
        mod = torch.zeros(T, dtype=torch.uint8, device="cuda")
        logits = torch.empty(T, E, device="cuda"); idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
        w = torch.empty(T, k, device="cuda"); cc = torch.empty((T + 63) // 64, E, 2, dtype=torch.int32, device="cuda")
        f = lambda: _lib.call("realb_router_topk_stats", x.data_ptr(), router.data_ptr(), None, mod.data_ptr(), T, H, E, k, 0, 1.0, 1e-12, logits.data_ptr(), idx.data_ptr(), w.data_ptr(), cc.data_ptr(), _lib.stream_ptr())
        for dbg in (0, 5):
            os.environ["REALB_DBG_ROUTER"] = str(dbg)
            for _ in range(3): f()
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                a.record(); f(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
            print(f"T={T:5d} H={H:5d} dbg={dbg} {sorted(ts)[5]*1e3:8.1f} us", flush=True)
# reference: an empty kernel-ish launch (torch fill) for launch overhead
y = torch.empty(64, device="cuda")
ts=[]
for _ in range(10):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); y.fill_(1.0); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print("torch fill_", sorted(ts)[5]*1e3, "us")
