"""Print the key ncu metrics (duration, DRAM, LSU/shared wavefronts, fp64 pipe,
occupancy, stall reasons) for every kernel in an .ncu-rep.

  python tools/ncu_kernel_metrics.py REPORT.ncu-rep [name-regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
filt = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
keys = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]
stall = [i for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
ki = h.index("Kernel Name")
for r in rows[2:]:
    if len(r) != len(h) or (filt and not filt.search(r[ki])):
        continue
    print(r[ki][:90])
    for k in keys:
        if k in h:
            print(f"   {k:70s} {r[h.index(k)]}")
    st = sorted(((float(r[i] or 0), h[i]) for i in stall), reverse=True)[:6]
    print("   top stalls:", ", ".join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, n in st))
