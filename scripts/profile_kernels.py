"""Launch each hot kernel on realistic shapes (for ncu -k regex:<name>).
Kimi-VL shapes: 1-GPU layer (8192 tokens) and the EP8 hot rank's FP4 GEMMs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
from paper_2604_19503_b200.policy import ClusterConfig, RealbParams
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

which = sys.argv[1] if len(sys.argv) > 1 else "layer"
shape = SHAPES["kimi"]
if which == "layer":
    T = 8192
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T))
    gu, dn = make_experts(shape)
    layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn, bias=torch.zeros(64, device="cuda")), max_tokens=T)
    for _ in range(3):
        layer.forward(x, mod, "baseline")
    torch.cuda.synchronize()
elif which == "ep8hot":
    # global EP8 batch; plan over 8 virtual ranks; run only the hot rank's experts (FP4 and BF16)
    T = 65536
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T))
    gu, dn = make_experts(shape)
    layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn, bias=torch.zeros(64, device="cuda")), max_tokens=T,
                     cluster=ClusterConfig(8, 1, 8, 1))
    res = layer.forward(x, mod, "realb", RealbParams())
    prec = res.plan.expert_precision(layer.placement).astype(np.int64)
    hot = sorted(res.plan.accelerated_ranks)[0]
    m = np.full(64, 2, np.int64); m[hot*8:(hot+1)*8] = 1
    for _ in range(3):
        layer.expert_compute(T, m)
    layer.quantize_experts(range(hot*8, (hot+1)*8))
    layer.forward(x, mod, "baseline")
    m[hot*8:(hot+1)*8] = 0
    for _ in range(3):
        layer.expert_compute(T, m)
    torch.cuda.synchronize()
print("done", which)
