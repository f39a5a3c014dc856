"""A/B: the 1-GPU Kimi layer with M = 64 MMAs on tail m-tiles (<= 64 valid rows; default)
vs M = 128 everywhere (REALB_DBG_BF16 bit 16), each its own layer + graph, interleaved
(bench_fp4.interleaved), twice each to expose the placement noise floor."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from bench_fp4 import interleaved
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
from paper_2604_19503_b200.policy import ClusterConfig
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

shape, T = SHAPES["kimi"], 8192
x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=8, rank=0))
gu, dn = make_experts(shape)
graphs = {}
for name, dbg in (("tail64_a", "0"), ("m128_a", "16"), ("tail64_b", "0"), ("m128_b", "16")):
    os.environ["REALB_DBG_BF16"] = dbg
    layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn), max_tokens=T,
                     cluster=ClusterConfig(1, 1, shape.num_experts, 1, False))
    graphs[name] = layer.capture(x, mod, "realb")
os.environ["REALB_DBG_BF16"] = "0"
torch.cuda.synchronize()
assert all(torch.equal(graphs["tail64_a"].y, g.y) for g in graphs.values())
with ClockSampler(0) as clk:
    res = interleaved({k: ({}, g.replay) for k, g in graphs.items()}, rounds=10, per=20)
out = {"ms": res, "clocks": clk.summary()}
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_tail64.json", "w"), indent=1)
