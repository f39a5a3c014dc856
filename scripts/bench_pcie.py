"""PCIe probe: H2D and D2H of one step's tensors (33.5 MB each), alone and
concurrently on separate streams, with pinned host memory."""
import torch, json
n = 8192 * 2048
xh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
yh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def h2d():
    with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): yh.copy_(yd, non_blocking=True)
def both():
    h2d(); d2h()
def syncall():
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
r = {}
r["h2d_ms"] = t(lambda: (h2d(), syncall()))
r["d2h_ms"] = t(lambda: (d2h(), syncall()))
r["both_ms"] = t(lambda: (both(), syncall()))
r["h2d_GBps"] = n * 2 / r["h2d_ms"] / 1e6
r["d2h_GBps"] = n * 2 / r["d2h_ms"] / 1e6
# chunked concurrent
def both_chunked(k=8):
    c = n // k
    for i in range(k):
        with torch.cuda.stream(s1): xd[i*c:(i+1)*c].copy_(xh[i*c:(i+1)*c], non_blocking=True)
        with torch.cuda.stream(s2): yh[i*c:(i+1)*c].copy_(yd[i*c:(i+1)*c], non_blocking=True)
r["both_chunked_ms"] = t(lambda: (both_chunked(), syncall()))
print(json.dumps(r))
