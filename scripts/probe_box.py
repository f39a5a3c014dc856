"""One-off box probe: device facts, library availability and a quantiser timing."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
out = {"device": torch.cuda.get_device_name(0), "cap": torch.cuda.get_device_capability(0),
       "sms": torch.cuda.get_device_properties(0).multi_processor_count,
       "cpu_count": os.cpu_count()}
try:
    out["lscpu"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines() if "Model name" in l]
except Exception as e:
    out["lscpu"] = str(e)
from paper_2604_19503_b200 import quant
w = torch.randn(16 * 2816, 2048, dtype=torch.bfloat16, device="cuda") * 0.02  # 16 experts gate_up
codes = torch.empty(w.shape[0], 1024, dtype=torch.uint8, device="cuda")
sf = torch.empty(w.numel() // 16, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for mc in (0, 74, 32):
    ts = []
    for i in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        quant.quantize_nvfp4(w, codes=codes, sf=sf, max_ctas=mc, check=False)
        b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts) // 2]
    out[f"quant_ms_maxctas{mc}"] = t
    out[f"quant_GBps_maxctas{mc}"] = w.numel() * 2.5625 / t / 1e6
# library probes
for name in ("_grouped_mm", "_scaled_grouped_mm", "_scaled_mm"):
    out[name] = hasattr(torch, name)
try:
    A = torch.randn(256, 2048, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(4, 2048, 512, device="cuda", dtype=torch.bfloat16)
    offs = torch.tensor([64, 128, 192, 256], device="cuda", dtype=torch.int32)
    torch._grouped_mm(A, B, offs=offs); out["grouped_mm_ok"] = True
except Exception as e:
    out["grouped_mm_ok"] = repr(e)[:200]
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
