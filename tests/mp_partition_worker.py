"""One rank of the multi-process partition test (tests/test_gpu_multiproc.py).

Launched by torch.distributed.run with FMV_NCCL_LIB pointing at the
host-staged NCCL test transport, so every rank can use cuda:0. torch.distributed
(gloo) only ships the 128-byte communicator id; all matvec collectives run
inside libfftmv_cuda (fmv_matvec_partitioned / fmv_matvec_partitioned_2d).
Writes this rank's outputs to <outdir>/rank<r>.npz.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2508_10202_b200 as F  # noqa: E402
from paper_2508_10202_b200 import _capi  # noqa: E402
from conftest import make_inputs  # noqa: E402

CFGS = ("ddddd", "dddds", "sdddd", "sssss", "hdddh")


def main():
    outdir, mode = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    nm, nd, nt = 64, 4, 32  # tests/golden/partition.npz shape (SPEC acceptance 8)
    col, m, d = make_inputs(F, nm, nd, nt)
    dims = F.ProblemDims(nm, nd, nt)
    ctx = F.Context(0)
    res = {}
    if mode == "1xp":
        grid = F.Grid1xP.split(world, nm)
        lo, hi = grid.shard_ranges[rank]
        shard = F.setup_operator(F.shard_operator(F.BlockColumn(dims, col), grid)[rank], ctx)
        dm = F.DistributedMatvec(dims, rank, world, shard=shard, transport="native", ctx=ctx)
        for cfg in CFGS:
            res[f"F_{cfg}"] = dm.forward(m[lo * nt:hi * nt], cfg)
            res[f"A_{cfg}"] = dm.adjoint(d if rank == 0 else None, cfg)
            # device-resident I/O through the same entry point
            res[f"Fdev_{cfg}"] = dm.forward(torch.from_numpy(m[lo * nt:hi * nt]).cuda(), cfg).cpu().numpy()
            res[f"Adev_{cfg}"] = dm.adjoint(torch.from_numpy(d).cuda(), cfg).cpu().numpy()
            # the async entry: F and F* enqueued back to back (two collectives in
            # flight on the stream), one fmv_synchronize for both
            xf = torch.from_numpy(m[lo * nt:hi * nt]).cuda()
            xa = torch.from_numpy(d).cuda()
            yf = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
            ya = torch.empty((hi - lo) * nt, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            L = _capi.lib()
            for kind, x, y in ((0, xf, yf), (1, xa, ya)):
                _capi.check(L.fmv_matvec_partitioned_async(ctx.handle, shard.handle, kind, cfg.encode(),
                                                           ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
            ctx.synchronize()
            res[f"Fasync_{cfg}"], res[f"Aasync_{cfg}"] = yf.cpu().numpy(), ya.cpu().numpy()
        out, t = dm.forward(m[lo * nt:hi * nt], "ddddd", times=True)
        res["F_times"] = np.array(list(t.phase_s) + [t.total_s])
        res["lohi"] = np.array([lo, hi])
        dm.close()
    elif mode == "2d":
        pr, pc = int(sys.argv[3]), int(sys.argv[4])
        g2 = F.GridPxQ.split(pr, pc, nd, nm)
        ri, cj = g2.coords(rank)
        (dlo, dhi), (mlo, mhi) = g2.row_ranges[ri], g2.col_ranges[cj]
        s2 = F.setup_operator(F.shard_operator_2d(F.BlockColumn(dims, col), g2)[rank], ctx)
        dm = F.DistributedMatvec2D(dims, pr, pc, rank, shard=s2, transport="native", ctx=ctx)
        for cfg in CFGS:
            res[f"F_{cfg}"] = dm.forward(m[mlo * nt:mhi * nt] if ri == 0 else None, cfg)
            res[f"A_{cfg}"] = dm.adjoint(d[dlo * nt:dhi * nt] if cj == 0 else None, cfg)
        res["rows"] = np.array([dlo, dhi])
        res["cols"] = np.array([mlo, mhi])
        dm.close()
    elif mode == "dead_peer":
        # rank 1 leaves after setup; rank 0's forward must fail (FMV_ENCCL), not hang
        grid = F.Grid1xP.split(world, nm)
        lo, hi = grid.shard_ranges[rank]
        shard = F.setup_operator(F.shard_operator(F.BlockColumn(dims, col), grid)[rank], ctx)
        dm = F.DistributedMatvec(dims, rank, world, shard=shard, transport="native", ctx=ctx)
        if rank == 0:
            try:
                dm.forward(m[lo * nt:hi * nt], "ddddd")
                res["error"] = np.array([0])
            except F.FmvError as e:
                res["error"] = np.array([1 if "[code 3]" in str(e) else 2])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
