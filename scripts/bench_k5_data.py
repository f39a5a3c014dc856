"""Why does K5 gate_up time differ between the bench layer and synthetic
operands? One run, burst timing (idle gap before each launch), four K5 cases
crossing {bench layout, uniform layout} x {bench data, randn data}, plus the
same-flops dense cuBLAS GEMM."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "scripts")]
import numpy as np, torch
from helpers import host_layout
from bench_fp4 import ev_time
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.clocks import ClockSampler
from paper_2604_19503_b200.moe import MoELayer
import bench as B


class A:
    config, tokens, vision_frac = "kimi", 8192, 0.7


torch.cuda.set_device(0)
shape, w, x, mod, cluster = B.build_layer(A, torch)
layer = MoELayer(w, max_tokens=8192, cluster=cluster)
layer.forward(x, mod, "baseline")
torch.cuda.synchronize()
E, H, I = 64, 2048, 1408
N, K = 2 * I, H
rows_cap = layer.rows_cap
lay_real = layer.layout.clone()
counts_real = layer.layout[8 + E:8 + 2 * E].cpu().numpy()
rng = np.random.default_rng(0)
cu = ((rng.random(E) * 0.4 + 0.8) * 768).astype(np.int64)
lay_u, rows_u = host_layout(cu, np.zeros(E, np.int64))
lay_u = torch.from_numpy(lay_u).cuda()
A_real = layer.a_bf16
A_rand = torch.randn(rows_cap, K, device="cuda").to(torch.bfloat16)
W_real = layer.w.w_gu
W_rand = (torch.randn(E * N, K, device="cuda") / K**0.5).to(torch.bfloat16)
o = torch.empty(rows_cap, N // 2, dtype=torch.bfloat16, device="cuda")
sp = _lib.stream_ptr()
pairs = 8192 * 6
ad = torch.randn(pairs, K, device="cuda").to(torch.bfloat16)
wd = (torch.randn(K, N, device="cuda") / K**0.5).to(torch.bfloat16)


def k5(a, w_, lay):
    return lambda: _lib.call("realb_grouped_gemm_bf16", a.data_ptr(), w_.data_ptr(), rows_cap, N, K, E,
                             lay.data_ptr(), 0, _lib.EPI_SWIGLU, o.data_ptr(), 0, sp)


# the same real rows with the 128-row padding rows (never read back) set to zero / randn
valid = torch.zeros(rows_cap, dtype=torch.bool, device="cuda")
lr = lay_real.cpu().numpy()
for e in range(E):
    valid[int(lr[8 + e]):int(lr[8 + e]) + int(lr[8 + E + e])] = True
A_padzero = A_real.clone()
A_padzero[~valid] = 0
A_padrand = A_real.clone()
A_padrand[~valid] = torch.randn(int((~valid).sum()), K, device="cuda").to(torch.bfloat16)
A_xlike = torch.randn(rows_cap, K, device="cuda").to(torch.bfloat16) * float(x.float().std())
vr = A_real[valid].float()
stats = {"valid_std": float(vr.std()), "valid_absmax": float(vr.abs().max()),
         "valid_zero_frac": float((vr == 0).float().mean()),
         "pad_nonfinite_frac": float((~torch.isfinite(A_real[~valid].float())).float().mean()),
         "x_std": float(x.float().std())}
v = {"real_padzero": k5(A_padzero, W_real, lay_real), "real_padrand": k5(A_padrand, W_real, lay_real),
     "randn_scaled_like_x": k5(A_xlike, W_real, lay_real),
     "real_layout_real_data": k5(A_real, W_real, lay_real), "real_layout_rand_A": k5(A_rand, W_real, lay_real),
     "real_layout_rand_W": k5(A_real, W_rand, lay_real), "real_layout_rand_both": k5(A_rand, W_rand, lay_real),
     "uniform_layout_rand_both": k5(A_rand, W_rand, lay_u), "cublas_dense": lambda: ad @ wd}
samples = {k: [] for k in v}
with ClockSampler(0) as clk:
    for _ in range(10):
        for k, f in v.items():
            torch.cuda.synchronize()
            time.sleep(0.01)
            samples[k].append(ev_time(f))
out = {k: float(np.median(s)) for k, s in samples.items()}
out["counts_real_minmax"] = [int(counts_real.min()), int(counts_real.max())]
out["stats"] = stats
out["w_real_std"] = float(W_real.float().std())
out["clocks"] = clk.summary()
print(json.dumps(out, indent=1))
