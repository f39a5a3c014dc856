"""BASELINE configs[4]: vision-token fraction and routing-skew sweep, ReaLB vs
all-BF16 EP, for the Kimi-VL / Qwen3-VL / ERNIE-4.5-VL(vision group) MoE-layer
shapes at EP 2/4/8 — virtual EP on one B200 (paper_2604_19503_b200/virtual_ep.py):
measured per-rank compute (compute-only speedup, engine.py:156) and the
projected full path (measured compute + K3, NVLink model for dispatch/combine).

  python scripts/sweep.py [--out gpurun_out/sweep.json] [--configs kimi,qwen,ernie_vision]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default="gpurun_out/sweep.json")
    p.add_argument("--configs", default="kimi,qwen,ernie_vision")
    p.add_argument("--ranks", default="2,4,8")
    p.add_argument("--vision", default="0.1,0.3,0.5,0.7,0.9")
    p.add_argument("--zipf", default="0.0,0.57,1.0,1.5")
    p.add_argument("--tokens", type=int, default=8192)
    a = p.parse_args()
    import torch

    from paper_2604_19503_b200.moe import SHAPES
    from paper_2604_19503_b200.virtual_ep import VirtualEP

    torch.cuda.set_device(0)
    rows = []
    t0 = time.time()
    for cfg in a.configs.split(","):
        isolated = SHAPES[cfg].modality_isolated
        # the ERNIE vision group only ever sees vision tokens (modality-split MoE):
        # its vision fraction is 1 by construction; only the skew is swept
        fvs = [1.0] if isolated else [float(v) for v in a.vision.split(",")]
        for R in [int(r) for r in a.ranks.split(",")]:
            vep = VirtualEP(torch, cfg, R, a.tokens)
            for zs in [float(z) for z in a.zipf.split(",")]:
                for fv in fvs:
                    r = vep.report(vision_frac=fv, zipf_s=zs)
                    rows.append(r)
                    print(f"{cfg:13s} R={R} zipf={zs:4.2f} fv={fv:.1f} imb={r['device_imbalance']:.2f} "
                          f"w4a4={r['plan_w4a4_ranks']} compute x{r['compute_only_speedup']:.2f} "
                          f"full x{r['projected_full_path_speedup']:.2f} "
                          f"(fp4-dispatch x{r['projected_full_path_speedup_fp4_dispatch']:.2f}) "
                          f"EP-layer x{r['projected_ep_layer_speedup']:.2f}/x{r['projected_ep_layer_speedup_fp4_dispatch']:.2f} "
                          f"text_exp={r['text_exposure']:.3f} [{time.time() - t0:.0f}s]", flush=True)
            del vep
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rows, f)


if __name__ == "__main__":
    main()
