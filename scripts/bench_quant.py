"""K3 microbenchmark: the hot rank's expert weights (Kimi EP8: 8 W4A4 experts'
gate_up + down) through realb_quantize_experts_nvfp4, L2 flushed between
launches, v1 / v2 / v3 (REALB_K3_VERSION) interleaved; achieved HBM GB/s on the
algorithmic bytes (2 B read + 0.5625 B written per weight) against two device
copies timed the same way: the same weights (read + write 2 B/weight) and a
copy moving the same total bytes as K3 (the "same-size copy")."""
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


def l2_flush():
    # read-only pass over 256 MB: L2 ends up holding CLEAN lines, so the timed kernel
    # pays no write-back of a previous flush's dirty lines (a zero_() flush leaves
    # ~126 MB dirty, written back inside the next timed launch)
    flush.sum()


def timed(f, reps=30):
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        l2_flush()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        f()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[reps // 2] / 1e3


out = {}
shapes = (("gate_up", wgu, 2 * I, H, cg, sg), ("down", wd, H, I, cd, sd))
VERS = ("v1", "v2", "v3")
res = {v: {n: [] for n, *_ in shapes} for v in VERS}
for rnd in range(5):
    for ver in VERS:
        os.environ["REALB_K3_VERSION"] = ver[1]
        for name, w, rpe, cols, c, s in shapes:
            f = lambda: _lib.call("realb_quantize_experts_nvfp4", w.data_ptr(), E, rpe, cols, prec.data_ptr(),
                                  c.data_ptr(), s.data_ptr(), flag.data_ptr(), 0, _lib.stream_ptr())
            res[ver][name].append(timed(f, 11))
os.environ.pop("REALB_K3_VERSION")
for ver in res:
    for name, w, rpe, cols, c, s in shapes:
        t = sorted(res[ver][name])[2]
        nbytes = 8 * rpe * cols * 2.5625
        out[f"k3_{ver}_{name}"] = dict(us=t * 1e6, GBps=nbytes / t / 1e9, algorithmic_bytes=nbytes)
# references: copies timed the same way
src = wgu[56 * 2 * I:]
dst = torch.empty_like(src)
t = timed(lambda: dst.copy_(src))
out["torch_copy_gate_up_hot"] = dict(us=t * 1e6, GBps=2 * src.numel() * 2 / t / 1e9)
nb = int(8 * 2 * I * H * 2.5625) // 2  # same total bytes as K3's gate_up: half read, half written
a8 = torch.empty(nb, dtype=torch.uint8, device="cuda")
b8 = torch.empty_like(a8)
t = timed(lambda: b8.copy_(a8))
out["same_size_copy_gate_up"] = dict(us=t * 1e6, GBps=2 * nb / t / 1e9)
for ver in VERS:
    out[f"k3_{ver}_gate_up"]["frac_of_same_size_copy"] = out["same_size_copy_gate_up"]["us"] / out[f"k3_{ver}_gate_up"]["us"]
# gate_up + down of the hot rank: one realb_quantize_experts2_nvfp4 launch vs the two
# single-matrix launches back to back; a copy moving the same total bytes beside them
os.environ["REALB_K3_VERSION"] = "2"
both = lambda: _lib.call("realb_quantize_experts2_nvfp4", wgu.data_ptr(), 2 * I, H, cg.data_ptr(), sg.data_ptr(),
                         wd.data_ptr(), H, I, cd.data_ptr(), sd.data_ptr(), E, prec.data_ptr(), flag.data_ptr(), 0,
                         _lib.stream_ptr())
def two():
    for name, w, rpe, cols, c, s in shapes:
        _lib.call("realb_quantize_experts_nvfp4", w.data_ptr(), E, rpe, cols, prec.data_ptr(), c.data_ptr(),
                  s.data_ptr(), flag.data_ptr(), 0, _lib.stream_ptr())
nb_all = int(8 * (2 * I * H + H * I) * 2.5625)
a_all = torch.empty(nb_all // 2, dtype=torch.uint8, device="cuda")
b_all = torch.empty_like(a_all)
tb, tt, tc = [], [], []
for rnd in range(5):
    tb.append(timed(both, 11)); tt.append(timed(two, 11)); tc.append(timed(lambda: b_all.copy_(a_all), 11))
tb, tt, tc = sorted(tb)[2], sorted(tt)[2], sorted(tc)[2]
out["k3_v2_gate_up_and_down_one_launch"] = dict(us=tb * 1e6, GBps=nb_all / tb / 1e9, algorithmic_bytes=nb_all,
                                                frac_of_same_size_copy=tc / tb)
out["k3_v2_gate_up_and_down_two_launches"] = dict(us=tt * 1e6, GBps=nb_all / tt / 1e9, frac_of_same_size_copy=tc / tt)
out["same_size_copy_gate_up_and_down"] = dict(us=tc * 1e6, GBps=nb_all / tc / 1e9)
# parity spot check v1 == v2 (bit-exact codes / scales)
outs = []
for ver in VERS:
    os.environ["REALB_K3_VERSION"] = ver[1]
    cg.zero_()
    sg.zero_()
    _lib.call("realb_quantize_experts_nvfp4", wgu.data_ptr(), E, 2 * I, H, prec.data_ptr(), cg.data_ptr(),
              sg.data_ptr(), flag.data_ptr(), 0, _lib.stream_ptr())
    outs.append((cg.clone(), sg.clone()))
out["all_versions_equal"] = all(torch.equal(outs[0][0], o[0]) and torch.equal(outs[0][1], o[1]) for o in outs[1:])
print(json.dumps(out, indent=1))
