"""K3 microbenchmark: the hot rank's expert weights (Kimi EP8: 8 experts gate_up + down)
through realb_quantize_experts_nvfp4, L2 flushed between launches; achieved HBM GB/s
on the algorithmic bytes (2 B read + 0.5625 B written per weight)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_19503_b200 import _lib
E, H, I = 64, 2048, 1408
wgu = (torch.randn(E * 2 * I, H, device="cuda") * 0.02).to(torch.bfloat16)
wd = (torch.randn(E * H, I, device="cuda") * 0.02).to(torch.bfloat16)
prec = torch.zeros(E, dtype=torch.uint8, device="cuda"); prec[56:] = 1
cg = torch.empty(E * 2 * I, H // 2, dtype=torch.uint8, device="cuda"); sg = torch.empty(E * 2 * I * H // 16, dtype=torch.uint8, device="cuda")
cd = torch.empty(E * H, I // 2, dtype=torch.uint8, device="cuda"); sd = torch.empty(E * H * I // 16, dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {}
for legacy in (False,):
  for name, w, rpe, cols, c, s in (("gate_up", wgu, 2 * I, H, cg, sg), ("down", wd, H, I, cd, sd)):
      name = "k3_" + name
      f = lambda: _lib.call("realb_quantize_experts_nvfp4", w.data_ptr(), E, rpe, cols, prec.data_ptr(), c.data_ptr(),
                            s.data_ptr(), flag.data_ptr(), 0, _lib.stream_ptr())
      for _ in range(3): f()
      ts = []
      for _ in range(20):
          flush.zero_()
          a, b = torch.cuda.Event(True), torch.cuda.Event(True)
          a.record(); f(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
      t = sorted(ts)[10] / 1e3
      nbytes = 8 * rpe * cols * 2.5625
      out[name] = dict(us=t * 1e6, GBps=nbytes / t / 1e9)
print(json.dumps(out))
# reference: a plain device copy of the same hot-rank weights (read + write), same flushing
src = wgu[56 * 2 * I:]
dst = torch.empty_like(src)
for _ in range(3): dst.copy_(src)
ts = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); dst.copy_(src); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
t = sorted(ts)[10] / 1e3
print(json.dumps({"torch_copy_gate_up_hot": dict(us=t * 1e6, GBps=2 * src.numel() * 2 / t / 1e9)}))
# read-only reduction of the same bytes (a read-bound reference)
ts = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); src.view(torch.int16).max(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
t = sorted(ts)[10] / 1e3
print(json.dumps({"torch_max_gate_up_hot": dict(us=t * 1e6, GBps=src.numel() * 2 / t / 1e9)}))
