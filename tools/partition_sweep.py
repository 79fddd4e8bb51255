"""f1, fp32-NCCL variants: the mixed-precision sweep over the PARTITIONED forward
matvec (sweep.hpp:74-119 run over forward_matvec_partitioned, partition.hpp:157-182)
at the C2 shape, with the exchange step's cost on B200.

On this one-GPU pool the p shards run in-process on cuda:0 (the library's
in-process partition: p shard pipelines, then the fixed left-balanced tree in
cfg[4]); errors are against the CPU reference's serial 'ddddd' F (oracle/_ref).
The exchange of a real p-GPU run is one all-gather of the p partial d's (Nd*Nt
values each, cfg[4] precision) plus the on-device tree; its time is modelled
from the message bytes at the NVLink 5 / NVSwitch rate (900 GB/s per direction
per GPU) plus a fixed per-collective latency, next to the measured shard step.

    python tools/partition_sweep.py [--p 8] [--out profiles/partition_sweep_r02]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MKL_NUM_THREADS", "1")
import numpy as np

import paper_2508_10202_b200 as F

NM, ND, NT, SEED = 5000, 100, 1000, 20250814
NVLINK_GBS = 900.0   # per direction per GPU (B200_PROFILING.md)
LAT_US = 10.0        # fixed cost per collective (assumed NCCL small-message latency on NVSwitch)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", default="2,8")
    ap.add_argument("--out", default="profiles/partition_sweep_r02")
    ap.add_argument("--render", help="only re-render the markdown from this json")
    a = ap.parse_args()
    if a.render:
        render(json.load(open(a.render)), a.out)
        return
    col = F.non_representable_fill(NM * ND * NT, F.seed_stream(SEED, 0))
    m = F.non_representable_fill(NM * NT, F.seed_stream(SEED, 1))
    dims = F.ProblemDims(NM, ND, NT)
    from oracle.oracle import have_ref, ref

    base = None
    if have_ref():
        R = ref()
        rop = R.setup_operator(NM, ND, NT, col)
        base = R.matvec(rop, 0, "ddddd", m)
        del rop
    rows = []
    for p in [int(v) for v in a.p.split(",")]:
        pop = F.setup_partitioned(F.BlockColumn(dims, col), F.Grid1xP.split(p, NM))
        for w in pop.workers:
            F.materialize_single(w)
        if base is None:
            base = F.forward_matvec_partitioned(pop, m, "ddddd").output.data
        # one rank's step: rank 0's shard pipeline, device-resident I/O, CUDA events (sweep.hpp timing loop)
        lo, hi = pop.grid.shard_ranges[0]
        shard_t = {r.config.render(): r.mean_s for r in F.preclab.sweep_operator(
            pop.workers[0], m[lo * NT:hi * NT], F.MatvecKind.Forward, 10, 2, timing="device")}
        for cfg in F.enumerate_configs():
            c = cfg.render()
            t0 = time.perf_counter()
            out = F.forward_matvec_partitioned(pop, m, c)
            wall = time.perf_counter() - t0
            err = F.relative_error(out.output.data, base)
            shard_ms = shard_t[c] * 1e3
            elem = 8 if c[4] == "d" else 4
            msg = ND * NT * elem
            comm_us = LAT_US + (p - 1) * msg / (NVLINK_GBS * 1e9) * 1e6
            rows.append({"p": p, "config": c, "rel_error": err, "shard_ms": shard_ms, "allgather_bytes_per_rank": msg,
                         "model_comm_us": comm_us, "comm_share": comm_us * 1e-3 / (shard_ms + comm_us * 1e-3),
                         # weak scaling (Nm = 5000 per GPU, the bench): the shard is the whole C2 operator, ~p x this one
                         "comm_share_weak": comm_us * 1e-3 / (p * shard_ms + comm_us * 1e-3),
                         "in_process_wall_ms": wall * 1e3})
        del pop
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    render(rows, a.out)


def render(rows, out):
    md = ["# f1: fp32-NCCL variants -- the Pareto sweep over the partitioned F at C2 (1 x B200, p shards in-process)",
          "",
          "Errors vs the CPU reference's serial `ddddd` F (oracle/_ref, non_representable_fill, seed 20250814). "
          "shard ms = one rank's shard matvec, device-resident I/O, CUDA events (mean of 10). The exchange (one all-gather of the p "
          f"partial d's, Nd*Nt = {ND * NT} values in cfg[4]) is modelled at {NVLINK_GBS:.0f} GB/s per direction "
          f"+ {LAT_US:.0f} us per collective.", ""]
    for p in sorted({r["p"] for r in rows}):
        md += [f"## p = {p}", "", "| config | rel error | shard ms | all-gather KB/rank | model comm us | comm share (C2 split p ways) "
               "| comm share (weak, Nm = 5000/GPU) |", "|---|---|---|---|---|---|---|"]
        for r in sorted([r for r in rows if r["p"] == p], key=lambda r: r["shard_ms"]):
            md.append(f"| {r['config']} | {r['rel_error']:.2e} | {r['shard_ms']:.3f} | {r['allgather_bytes_per_rank'] / 1e3:.0f} "
                      f"| {r['model_comm_us']:.1f} | {100 * r['comm_share']:.2f}% | {100 * r['comm_share_weak']:.2f}% |")
        md.append("")
    dd = {r["p"]: r for r in rows if r["config"] == "dssdd"}
    ds = {r["p"]: r for r in rows if r["config"] == "dssds"}
    pmax = max(dd)
    a_, b_ = dd[pmax], ds[pmax]
    md += [f"Reading: the fp32 reduce (`dssds` vs `dssdd`) halves the message. At p = {pmax}: "
           f"{a_['model_comm_us']:.1f} -> {b_['model_comm_us']:.1f} us for an error of {a_['rel_error']:.2e} -> "
           f"{b_['rel_error']:.2e}; that is {100 * (a_['comm_share'] - b_['comm_share']):.1f} % of the step with C2 split "
           f"{pmax} ways (exchange share {100 * a_['comm_share']:.1f} % -> {100 * b_['comm_share']:.1f} %) and "
           f"{100 * (a_['comm_share_weak'] - b_['comm_share_weak']):.2f} % weak-scaled (Nm = 5000/GPU, the bench). "
           "Within one 8 x B200 NVSwitch node the trade-off is worth a few microseconds; the paper's win (PAPER.md:152, "
           ">= 512 GPUs on Frontier) comes from exchange costs this node does not have."]
    open(out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
