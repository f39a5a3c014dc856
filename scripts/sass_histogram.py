"""Per-kernel SASS instruction histogram of the built C-ABI library (evidence that
the hot kernels are tcgen05 / TMA / TMEM native): cuobjdump -sass on
paper_2604_19503_b200/lib/librealb_b200.so, opcode counts per kernel for the
instruction families that matter (tensor-core MMAs, TMA loads / stores, TMEM
loads and copies, bulk copies, FP4 / E4M3 conversions, packed FP32), plus the
ptxas resource usage (registers, spills, shared memory).

  python scripts/sass_histogram.py  -> profiles/r02/sass_histogram.json
"""
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_19503_b200", "lib", "librealb_b200.so")
FAMILIES = ["UTCHMMA", "UTCOMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "UTCCP",
            "UTCBAR", "SYNCS", "F2FP", "FFMA2", "FMUL2", "FADD2", "LDG", "STG", "LDS", "STS", "ELECT", "R2UR"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
        return out.strip().split("\n")
    except Exception:  # noqa: BLE001
        return names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m and cur:
            op = m.group(2)
            base = op.split(".")[0]
            kernels[cur][base] += 1
            if base in ("F2FP", "UTCHMMA", "UTCOMMA", "UTMALDG", "UTMASTG", "UTCCP", "LDTM"):
                kernels[cur][op] += 1
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    usage = {}
    for fn, u in re.findall(r"Function (\S+):\s*\n\s*(REG:.*)", res):
        usage[fn] = dict(re.findall(r"(\w+(?:\[\d\])?):(\d+)", u))
    names = list(kernels)
    pretty = demangle(names)
    out = {}
    for n, p in zip(names, pretty):
        c = kernels[n]
        fam = {k: v for k, v in sorted(c.items()) if k.split(".")[0] in FAMILIES}
        out[p] = {"total_instructions": sum(v for k, v in c.items() if "." not in k or k.split(".")[0] not in
                                            ("F2FP", "UTCHMMA", "UTCOMMA", "UTMALDG", "UTMASTG", "UTCCP", "LDTM")),
                  "families": fam, "resources": usage.get(n, {})}
    summary = Counter()
    for v in out.values():
        for k, n in v["families"].items():
            summary[k] += n
    doc = {"library": os.path.relpath(LIB, ROOT), "kernels": out, "library_totals": dict(sorted(summary.items())),
           "how": "cuobjdump -sass / -res-usage of the built sm_100a library; opcode counts per kernel"}
    dst = os.path.join(ROOT, "profiles", "r02", "sass_histogram.json")
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    json.dump(doc, open(dst, "w"), indent=1)
    print(json.dumps({k: v for k, v in doc["library_totals"].items() if k.startswith(("UT", "LDTM", "F2FP"))}, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
