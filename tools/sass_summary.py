#!/usr/bin/env python3
"""Instruction-class counts per kernel in libqtng.so's SASS (cuobjdump), the
static "tell" of what each kernel uses: FP64 pipe (DMUL/DADD/DFMA), tensor
cores (DMMA, UTC*), TMA / bulk async copies (UTMALDG, UBLKCP, SYNCS), loads."""
import collections, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2204_06045_b200", "libqtng.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
CLASSES = ["DMUL", "DADD", "DFMA", "DMMA", "UTCHMMA", "UTCQMMA", "UTCIMMA", "LDTM", "STTM",
           "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "LDG", "LDS", "STG", "STS", "LDL", "STL", "SHFL",
           "ATOMG", "RED"]
per = collections.OrderedDict()
name = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        per.setdefault(name, collections.Counter())
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and name:
        op = m.group(2)
        for c in CLASSES:
            if op == c or op.startswith(c + "."):
                per[name][c] += 1
                break
        per[name]["total"] += 1
def short(n):
    n = re.sub(r"_ZN4qtng\d+c(128|64)\d+_GLOBAL__N__[0-9a-f_]+?_kernels_cu_[0-9a-f]+", r"c\1::", n)
    return n[:70]
print("kernel".ljust(72), " ".join(c.rjust(7) for c in ["total"] + CLASSES))
for n, c in per.items():
    if "kernel" not in n and "Kernel" not in n:
        continue
    print(short(n).ljust(72), " ".join(str(c.get(k, 0)).rjust(7) for k in ["total"] + CLASSES))
