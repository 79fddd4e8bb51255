"""Top SASS lines by warp-stall samples for one kernel of an .ncu-rep (source page).

  python tools/ncu_hotspots.py REPORT.ncu-rep KERNEL_BASE_NAME [N] [LAUNCH_SKIP]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kre, "--launch-skip", skip,
                      "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
name = lines[0]
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si, ni, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
data = [(int(r[si] or 0), r[ni].strip(), int(r[ei] or 0)) for r in rows[1:]
        if len(r) == len(h) and r[0].startswith("0x")]
tot = sum(d[0] for d in data) or 1
print(name.replace('"Kernel Name",', "").strip('",'))
print(f"{'stall %':>7}  {'inst exec':>10}  SASS")
for s, src, e in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / tot:6.1f}%  {e:10d}  {src}")
