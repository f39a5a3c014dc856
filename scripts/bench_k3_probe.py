"""K3 timing probes (REALB_DBG_K3): the one-launch K3 over the Kimi EP8 hot rank's
weights (8 experts' gate_up + down) as shipped (0), with its stores but no
conversion (1), and with its loads only (2), beside a device copy moving the same
bytes; L2 cleaned between launches, interleaved rounds, median."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19503_b200 import _lib  # noqa: E402

E, H, I = 64, 2048, 1408
wgu = (torch.randn(E * 2 * I, H, device="cuda") * 0.02).to(torch.bfloat16)
wd = (torch.randn(E * H, I, device="cuda") * 0.02).to(torch.bfloat16)
prec = torch.zeros(E, dtype=torch.uint8, device="cuda")
prec[56:] = 1
cg = torch.empty(E * 2 * I, H // 2, dtype=torch.uint8, device="cuda")
sg = torch.empty(E * 2 * I * H // 16, dtype=torch.uint8, device="cuda")
cd = torch.empty(E * H, I // 2, dtype=torch.uint8, device="cuda")
sd = torch.empty(E * H * I // 16, dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
nb = int(8 * (2 * I * H + H * I) * 2.5625)
a8 = torch.empty(nb // 2, dtype=torch.uint8, device="cuda")
b8 = torch.empty_like(a8)
rd = torch.empty(8 * (2 * I * H + H * I) * 2 // 4, dtype=torch.float32, device="cuda")


def k3():
    _lib.call("realb_quantize_experts2_nvfp4", wgu.data_ptr(), 2 * I, H, cg.data_ptr(), sg.data_ptr(),
              wd.data_ptr(), H, I, cd.data_ptr(), sd.data_ptr(), E, prec.data_ptr(), flag.data_ptr(), 0,
              _lib.stream_ptr())


def timed(f):
    flush.sum()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); f(); b.record(); b.synchronize()
    return a.elapsed_time(b) * 1e3


res = {}
variants = {"k3": ("0", k3), "k3_no_conversion": ("1", k3), "k3_loads_only": ("2", k3),
            "copy_same_bytes": (None, lambda: b8.copy_(a8)), "read_weights_sum": (None, lambda: rd.sum())}
for rnd in range(15):
    for name, (dbg, f) in variants.items():
        if dbg is not None:
            os.environ["REALB_DBG_K3"] = dbg
        if rnd == 0:
            f(); f()
        res.setdefault(name, []).append(timed(f))
os.environ.pop("REALB_DBG_K3", None)
out = {k: sorted(v)[len(v) // 2] for k, v in res.items()}
out["algorithmic_bytes"] = nb
out["k3_GBps"] = nb / out["k3"] / 1e3
print(json.dumps(out, indent=1))
