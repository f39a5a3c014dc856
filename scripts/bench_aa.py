"""Methodology check for the interleaved layer A/B benchmarks: several MoE layers
with identical settings (and some with another dispatch mode), each its own
buffers and CUDA graph, timed interleaved. Any spread between identical layers
is placement / ordering bias, the noise floor of the A/B comparisons.

  python scripts/bench_aa.py [--modes copy,copy,copyin,copyin]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from bench_fp4 import interleaved
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
from paper_2604_19503_b200.policy import ClusterConfig
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

p = argparse.ArgumentParser()
p.add_argument("--modes", default="copy,copy,copyin,copyin,copy")
a = p.parse_args()
shape, T = SHAPES["kimi"], 8192
x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=1, rank=0))
gu, dn = make_experts(shape)
graphs = {}
for i, m in enumerate(a.modes.split(",")):
    layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn), max_tokens=T,
                     cluster=ClusterConfig(1, 1, shape.num_experts, 1, False))
    layer.dispatch_mode = m
    graphs[f"{i}_{m}"] = layer.capture(x, mod, "realb")
torch.cuda.synchronize()
with ClockSampler(0) as clk:
    res = interleaved({k: ({}, g.replay) for k, g in graphs.items()}, rounds=10, per=10)
out = {"ms": res, "clocks": clk.summary()}
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/bench_aa.json", "w"), indent=1)
