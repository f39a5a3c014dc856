"""A/B/C: the single-GPU layer with copy dispatch (realb_dispatch_permute + K5 on
the grouped operand), gather dispatch (realb_dispatch_index + K5 reading x rows
with cp.async loaders) and copy-in dispatch (realb_dispatch_index + K5 whose
spare warps copy the rows while its mainloop runs), each captured as one CUDA graph, timed interleaved
(bench_fp4.interleaved, L2 not flushed) with NVML clocks; plus the two gate_up
kernels alone.

  python scripts/bench_dispatch.py [--config kimi] [--tokens 8192]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="kimi")
    p.add_argument("--tokens", type=int, default=8192)
    a = p.parse_args()
    import torch

    from bench_fp4 import interleaved
    from paper_2604_19503_b200 import _lib
    from paper_2604_19503_b200.clocks import ClockSampler
    from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
    from paper_2604_19503_b200.policy import ClusterConfig
    from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

    torch.cuda.set_device(0)
    shape = SHAPES[a.config]
    T = a.tokens
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=1, rank=0), device="cuda")
    gu, dn = make_experts(shape, device="cuda")
    layers, graphs = {}, {}
    for mode in ("copy", "gather", "copyin"):
        layer = MoELayer(MoEWeights.from_hf(shape, router, gu, dn), max_tokens=T,
                         cluster=ClusterConfig(1, 1, shape.num_experts, 1, shape.modality_isolated))
        layer.dispatch_mode = mode
        layers[mode] = layer
        graphs[mode] = layer.capture(x, mod, "realb")
    torch.cuda.synchronize()
    assert torch.equal(graphs["copy"].y, graphs["gather"].y) and torch.equal(graphs["copy"].y, graphs["copyin"].y)
    sp = _lib.stream_ptr()
    variants = {f"layer_{m}": ({}, graphs[m].replay) for m in graphs}
    for m, layer in layers.items():
        variants[f"gate_up_{m}"] = ({}, lambda layer=layer: layer._gate_up_bf16(layer.layout.data_ptr(), sp,
                                                                                 in_forward=True))
    with ClockSampler(0) as clk:
        res = interleaved(variants)
    out = {"config": a.config, "tokens": T, "ms": res, "clocks": clk.summary()}
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/bench_dispatch.json", "w"), indent=1)


if __name__ == "__main__":
    main()
