"""Summarise an ncu source page (SASS) by hottest instructions:
    python tools/ncu_sass.py rep.ncu-rep BASE_NAME_REGEX SKIP [N]   (SKIP = index among matching launches)"""
import csv, io, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + rx, "--launch-skip", str(skip), "--launch-count", "1"],
                     stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
body = [r for r in rows[hdr + 1:] if len(r) == len(h) and r[0] != "Address"]
si, ei, smp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot_e = sum(float(r[ei] or 0) for r in body)
tot_s = sum(float(r[smp] or 0) for r in body)
print(rows[0][:2], "instructions", tot_e, "samples", tot_s)
# opcode histogram
from collections import Counter
c = Counter()
for r in body:
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    c[op.split(".")[0]] += float(r[ei] or 0)
print("opcode mix:", [(k, round(v / tot_e * 100, 1)) for k, v in c.most_common(15)])
body.sort(key=lambda r: -float(r[smp] or 0))
for r in body[:n]:
    print(f"{float(r[smp] or 0) / tot_s * 100:5.1f}% smp  {float(r[ei] or 0):12.0f} exec  {r[si].strip()[:90]}")
