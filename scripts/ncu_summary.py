"""Summarise ncu --set full reports into profiles/<round>/ncu_summary.json and
profiles/traffic.json (per-launch DRAM bytes of the bench's roofline kernel)."""
import csv, io, json, subprocess, sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "second": 1}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * UNIT.get(units[i], 1) if units[i] in UNIT else v
        t = d.get("gpu__time_duration.sum")
        rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
        if t:
            d["dram_TBps"] = (rd + wr) / t / 1e12
        out.append(d)
    return out


if __name__ == "__main__":
    rnd = sys.argv[1]
    reps = sys.argv[2:]
    summ = {Path(r).stem: summarise(r) for r in reps}
    Path(f"profiles/{rnd}").mkdir(parents=True, exist_ok=True)
    Path(f"profiles/{rnd}/ncu_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
    tf = Path("profiles/traffic.json")
    traffic = json.loads(tf.read_text()) if tf.exists() else {}
    for name, ks in summ.items():
        for d in ks:
            if "grouped_gemm_bf16_kernel<256, 4, 1" in d["kernel"] and name.startswith("prof_layer"):
                traffic["gate_up_kimi_8192"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tf.write_text(json.dumps(traffic, indent=1) + "\n")
    print(json.dumps(summ, indent=1)[:3000])
