"""Registers / stack / shared per kernel of a libgsb build: python scripts/resusage.py [so] [filter]"""
import re, subprocess, sys
so = sys.argv[1] if len(sys.argv) > 1 else "paper_2406_06022_b200/libgsb.so"
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True, text=True).stdout.splitlines()
names = []
for i, l in enumerate(out):
    m = re.match(r"\s*Function (\S+):", l)
    if m and i + 1 < len(out):
        r = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", out[i + 1])
        if r:
            names.append((m.group(1), r.groups()))
dm = subprocess.run(["c++filt"], input="\n".join(n for n, _ in names), capture_output=True, text=True).stdout.splitlines()
for d, (_, (reg, st, sh)) in zip(dm, names):
    short = re.sub(r"\(.*", "", d)
    if flt in short:
        print(f"{reg:>4} {st:>4} {sh:>6}  {short}")
