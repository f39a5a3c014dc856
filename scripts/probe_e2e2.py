"""e2e pipeline timeline: per-step events on the H2D / compute / D2H streams."""
import os, sys, json, types
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2604_19503_b200.moe import MoELayer
from paper_2604_19503_b200.policy import RealbParams

args = types.SimpleNamespace(config="kimi", tokens=8192, vision_frac=0.7, steps=20, warmup=5)
torch.cuda.set_device(0)
shape, w, x, mod, cluster = bench.build_layer(args, torch)
layer = MoELayer(w, max_tokens=8192, cluster=cluster)
T, H = x.shape
nbuf, n = 2, 25
xs = [torch.empty_like(x) for _ in range(nbuf)]; ms = [torch.empty_like(mod) for _ in range(nbuf)]
ys = [torch.empty(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(nbuf)]
for i in range(nbuf): xs[i].copy_(x); ms[i].copy_(mod)
graphs = [layer.capture(xs[i], ms[i], "realb", RealbParams(), out=ys[i]) for i in range(nbuf)]
xh = [x.cpu().pin_memory() for _ in range(4)]; mh = [mod.cpu().pin_memory() for _ in range(4)]
yh = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
comp = torch.cuda.current_stream(); up, down = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
hs, he, cs, ce, ds, de = ([E() for _ in range(n)] for _ in range(6))
torch.cuda.synchronize()
base = E(); base.record(); 
for i in range(n):
    b = i % nbuf
    with torch.cuda.stream(up):
        if i >= nbuf: up.wait_event(ce[i - nbuf])
        hs[i].record(up)
        xs[b].copy_(xh[i % 4], non_blocking=True); ms[b].copy_(mh[i % 4], non_blocking=True)
        he[i].record(up)
    comp.wait_event(he[i])
    if i >= nbuf: comp.wait_event(de[i - nbuf])
    cs[i].record(comp); graphs[b].replay(); ce[i].record(comp)
    with torch.cuda.stream(down):
        down.wait_event(ce[i]); ds[i].record(down)
        yh[i % 4].copy_(ys[b], non_blocking=True); de[i].record(down)
torch.cuda.synchronize()
f = lambda e: base.elapsed_time(e)
rows = [[round(f(a[i]), 3) for a in (hs, he, cs, ce, ds, de)] for i in range(n)]
for i in range(0, 9): print(i, rows[i], "h2d", round(rows[i][1]-rows[i][0],3))
print("per-step compute start delta:", np.diff([r[2] for r in rows[5:]]).round(3).tolist())
print("compute dur:", [round(r[3] - r[2], 3) for r in rows[5:12]], "h2d dur:", [round(r[1] - r[0], 3) for r in rows[5:12]],
      "d2h dur:", [round(r[5] - r[4], 3) for r in rows[5:12]])
