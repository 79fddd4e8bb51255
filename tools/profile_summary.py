"""Summarise ncu captures into profiles/ (committed evidence).

  python tools/profile_summary.py ROUND LAUNCH_CSV FULL_REP [BENCH_JSON]

Writes profiles/ncu_launches_<round>.csv (copy), profiles/ncu_summary.json
(per-kernel duration / DRAM bytes / throughput; bench.py reads
sbgemv_dram_bytes_per_launch from it) and profiles/ncu_summary_<round>.md.
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, launch_csv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
bench = sys.argv[4] if len(sys.argv) > 4 else None
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)
shutil.copy(launch_csv, os.path.join(prof, f"ncu_launches_{rnd}.csv"))

rows = list(csv.reader(open(launch_csv)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
launches = [(r[ki], float(r[vi])) for r in rows[hi + 1:] if len(r) == len(h)]
# drop the one-time operator setup (every launch before the first SBGEMV except the
# matvec's own r2c right before it)
first = next(i for i, (n, _) in enumerate(launches) if "k_sbgemv" in n)
launches = launches[max(0, first - 1):]


def short(n):
    return n.split("(")[0].replace("void ", "").strip()


tot = {}
for n, v in launches:
    k = short(n)
    tot.setdefault(k, [0, 0.0])
    tot[k][0] += 1
    tot[k][1] += v

out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                     text=True).stdout
raw = list(csv.reader(io.StringIO(out)))
rh = raw[0]
units = raw[1]


def col(name):
    return rh.index(name) if name in rh else None


want = {
    "time": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed", "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size", "block": "launch__block_size", "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
kern = []
for r in raw[2:]:
    d = {"name": r[rh.index("Kernel Name")]}
    for k, m in want.items():
        c = col(m)
        if c is None:
            continue
        v = r[c].replace(",", "")
        try:
            d[k] = float(v) * scale.get(units[c], 1)
        except ValueError:
            d[k] = v
    kern.append(d)

summary = {"round": rnd, "launch_totals_ns": {k: {"launches": n, "total_ns": t} for k, (n, t) in tot.items()},
           "full_capture": kern}
gemv = [k for k in kern if "k_sbgemv" in k["name"]]
if gemv:
    summary["sbgemv_dram_bytes_per_launch"] = sum(k.get("rd", 0) + k.get("wr", 0) for k in gemv) / len(gemv)
json.dump(summary, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=1)

md = [f"# ncu summary, {rnd}", "", "Command: `ncu --metrics gpu__time_duration.sum --clock-control none` "
      "(launch list, operator setup excluded) and `ncu --set full --clock-control none --import-source on` (full capture) on "
      "`python tools/profile_step.py` (C2 operator, 4 x (F + F*), cold-cache serialised launches).", "",
      "## Launch list (share of device time)", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
allt = sum(t for _, t in tot.values())
for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    md.append(f"| `{k}` | {n} | {t / 1e3:.1f} | {t / allt * 100:.1f}% |")
md += ["", "## Full capture (one launch each)", "",
       "| kernel | grid x block | regs | time us | DRAM read MB | DRAM write MB | DRAM % peak | SM % | achieved GB/s (DRAM) |",
       "|---|---|---|---|---|---|---|---|---|"]
for k in kern:
    t = k.get("time", 0)
    gbs = (k.get("rd", 0) + k.get("wr", 0)) / t / 1e9 if t else 0
    md.append(f"| `{short(k['name'])[:70]}` | {k.get('grid', 0):.0f} x {k.get('block', 0):.0f} | {k.get('regs', 0):.0f} | "
              f"{t * 1e6:.1f} | {k.get('rd', 0) / 1e6:.1f} | {k.get('wr', 0) / 1e6:.1f} | {k.get('dram_pct', 0):.1f} | "
              f"{k.get('sm_pct', 0):.1f} | {gbs:.0f} |")
if bench:
    md += ["", "## bench.py line (same build)", "", "```", open(bench).read().strip(), "```"]
open(os.path.join(prof, f"ncu_summary_{rnd}.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
