"""Per-kernel SASS instruction counts of the product library (dev tool):
    python tools/sass_summary.py > profiles/r02/sass_summary.md"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1401_2720_b200" / "_lib" / "libjhsvd_b200.so"
OPS = ("DMMA", "UTMALDG", "UBLKCP", "DFMA", "LDGSTS", "SYNCS", "MUFU")


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    counts = collections.OrderedDict()
    name = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = m.group(1)
            counts[name] = collections.Counter()
            continue
        if name is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if not m:
            continue
        op, suf = m.group(1), m.group(2) or ""
        if op == "MUFU" and ".64" not in suf and "64H" not in suf:
            continue
        for o in OPS:
            if op == o:
                counts[name][o] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True,
                               text=True).stdout.splitlines()
    print("# SASS instruction summary of the product library (round 2 head)\n")
    print("`cuobjdump -sass paper_1401_2720_b200/_lib/libjhsvd_b200.so`, counted per kernel "
          "(static instructions; tools/sass_summary.py).")
    print("DMMA = `mma.sync.m8n8k4.f64` (FP64 tensor core), UBLKCP = `cp.async.bulk` (TMA engine "
          "bulk copy), UTMALDG = `cp.async.bulk.tensor` (TMA tensor tile), LDGSTS = `cp.async`, SYNCS = mbarrier operations, MUFU = FP64 reciprocal / "
          "rsqrt seeds of the IEEE division / sqrt paths.\n")
    print("| DMMA | UTMALDG | UBLKCP | DFMA | LDGSTS | SYNCS | MUFU64 | kernel |")
    print("|---|---|---|---|---|---|---|---|")
    rows = sorted(zip(demangled, counts.values()), key=lambda r: -r[1]["DMMA"])
    for dn, c in rows:
        dn = re.sub(r"\(.*", "", dn.replace("(anonymous namespace)::", ""))
        print(f"| {c['DMMA']} | {c['UTMALDG']} | {c['UBLKCP']} | {c['DFMA']} | {c['LDGSTS']} | "
              f"{c['SYNCS']} | "
              f"{c['MUFU']} | `{dn}` |")


if __name__ == "__main__":
    main()
