"""SASS instruction census of libltb.so: per kernel, the tcgen05 / TMA / tensor-memory and
FP64-matrix instructions that prove which hardware paths the build uses
(UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM / STTM = tcgen05.ld / st, UTMALDG /
UTMASTG = TMA tensor load / store, DMMA = FP64 tensor MMA, FFMA2 / DFMA = vector FP32 / FP64 FMA).
Usage: python tools/sass_census.py [libltb.so] > profiles/rNN_sass_census.md"""
import re
import subprocess
import sys
from collections import Counter, defaultdict

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2202_02870_b200/libltb.so"
ops = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "DMMA", "HMMA", "FFMA2", "DFMA", "MUFU"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
cur, counts = None, defaultdict(Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m:
        op = m.group(1).split(".")[0]
        if op in ops:
            counts[cur][op] += 1


def short(name: str) -> str:
    try:
        d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        d = name
    d = re.sub(r"\(anonymous namespace\)::", "", d)
    return d.split("(")[0][:90]


tot = Counter()
print(f"# SASS census of `{lib}`\n")
print("| kernel | " + " | ".join(ops) + " |")
print("|---|" + "---|" * len(ops))
for k in sorted(counts, key=lambda k: -sum(counts[k][o] for o in ops[:6])):
    c = counts[k]
    if not any(c[o] for o in ops):
        continue
    tot.update(c)
    print(f"| `{short(k)}` | " + " | ".join(str(c[o]) for o in ops) + " |")
print("| **total** | " + " | ".join(str(tot[o]) for o in ops) + " |")
