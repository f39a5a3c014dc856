"""Launch the router alone (Kimi shape, T tokens) for an ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.moe import SHAPES
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
shape = SHAPES["kimi"]
x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T))
E, k, H = 64, 6, 2048
logits = torch.empty(T, E, device="cuda"); idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
w = torch.empty(T, k, device="cuda"); cc = torch.empty((T + 63) // 64, E, 2, dtype=torch.int32, device="cuda")
bias = torch.zeros(E, device="cuda")
for _ in range(3):
    _lib.call("realb_router_topk_stats", x.data_ptr(), router.data_ptr(), bias.data_ptr(), mod.data_ptr(), T, H, E, k,
              shape.scoring, shape.routed_scaling, 1e-12, logits.data_ptr(), idx.data_ptr(), w.data_ptr(), cc.data_ptr(),
              _lib.stream_ptr())
torch.cuda.synchronize()
print("ok")
