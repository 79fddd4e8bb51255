"""Multi-rank check of the native NCCL path (fmv_matvec_partitioned and the 2-D
grid), launched with torch.distributed.run --nproc-per-node N: rank r uses GPU
r % device_count and holds its Grid1xP shard; every rank checks the distributed
F / F* against the serial matvec of the full operator. On a one-GPU box NCCL
refuses two ranks on one device ("Duplicate GPU detected"), which the script
reports through the library's FMV_ENCCL error."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2508_10202_b200 as F

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(dev)
dist.init_process_group("gloo")  # id exchange only; the matvec collectives run in the library's NCCL comm
nm, nd, nt = 64, 6, 50
col = F.uniform_fill(nm * nd * nt, 1)
m = F.uniform_fill(nm * nt, 2)
d = F.uniform_fill(nd * nt, 3)
dims = F.ProblemDims(nm, nd, nt)
grid = F.Grid1xP.split(world, nm)
lo, hi = grid.shard_ranges[rank]
ctx = F.Context(dev)
shard = F.setup_operator(F.shard_operator(F.BlockColumn(dims, col), grid)[rank], ctx)
try:
    dm = F.DistributedMatvec(dims, rank, world, shard=shard, transport="native")
except Exception as e:
    print(f"rank {rank}: NCCL init failed: {e}", flush=True)
    sys.exit(0)
serial = F.setup_operator(F.BlockColumn(dims, col), ctx)
ok = True
for cfg in ("ddddd", "dddds", "sdddd"):
    fd = dm.forward(m[lo * nt:hi * nt], cfg)
    am = dm.adjoint(d if rank == 0 else None, cfg)
    sf = F.forward_matvec(serial, m, cfg).output.data
    sa = F.adjoint_matvec(serial, d, cfg).output.data
    ef = float(np.linalg.norm(fd - sf) / np.linalg.norm(sf))
    ea = float(np.linalg.norm(am - sa[lo * nt:hi * nt]) / np.linalg.norm(sa[lo * nt:hi * nt]))
    tol = 1e-12 if cfg == "ddddd" else 1e-6
    ok &= ef <= tol and ea <= tol
    print(f"rank {rank} {cfg}: F rel err {ef:.2e}, F* slice rel err {ea:.2e}", flush=True)
dm.close()
g2 = F.GridPxQ.split(2, 1, nd, nm) if world == 2 else None
if g2 is not None:
    ri, cj = g2.coords(rank)
    (dlo, dhi), (mlo, mhi) = g2.row_ranges[ri], g2.col_ranges[cj]
    s2 = F.setup_operator(F.shard_operator_2d(F.BlockColumn(dims, col), g2)[rank], ctx)
    d2 = F.DistributedMatvec2D(dims, 2, 1, rank, shard=s2, transport="native")
    fd = d2.forward(m if ri == 0 else None)
    sf = F.forward_matvec(serial, m).output.data[dlo * nt:dhi * nt]
    e2 = float(np.linalg.norm(fd - sf) / np.linalg.norm(sf))
    ok &= e2 <= 1e-12
    print(f"rank {rank} 2x1 grid: F rows rel err {e2:.2e}", flush=True)
    d2.close()
print(f"rank {rank}: {'OK' if ok else 'FAIL'}", flush=True)
dist.destroy_process_group()
