"""e2e pipeline probe: graph replay alone vs the double-buffered H2D/compute/D2H
pipeline of bench.run_e2e, and variants without one of the transfers."""
import os, sys, json, types
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2604_19503_b200.moe import MoELayer
from paper_2604_19503_b200.policy import RealbParams

args = types.SimpleNamespace(config="kimi", tokens=8192, vision_frac=0.7, steps=20, warmup=5)
torch.cuda.set_device(0)
shape, w, x, mod, cluster = bench.build_layer(args, torch)
layer = MoELayer(w, max_tokens=8192, cluster=cluster)
g = layer.capture(x, mod, "realb", RealbParams())
def t(fn, reps=20):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
r = {"graph_back_to_back_ms": t(g.replay)}
ms, _ = bench.run_e2e(torch, layer, x, mod, RealbParams(), args)
r["e2e_ms"] = ms
print(json.dumps(r))
# compute while PCIe copies stream concurrently on other streams
n = x.numel()
xh = x.cpu().pin_memory(); yh = torch.empty(8192 * shape.hidden, dtype=torch.bfloat16).pin_memory()
xd = torch.empty_like(x); yd = torch.empty(8192 * shape.hidden, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def g_with_copies():
    with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2): yh.copy_(yd, non_blocking=True)
    g.replay()
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
r2 = {"graph_plus_concurrent_copies_ms": t(g_with_copies)}
# host enqueue cost of one e2e iteration (no GPU wait)
import time
torch.cuda.synchronize()
h0 = time.perf_counter()
for _ in range(20):
    g.replay()
h1 = time.perf_counter()
torch.cuda.synchronize()
r2["host_replay_enqueue_ms"] = (h1 - h0) / 20 * 1e3
print(json.dumps(r2))
