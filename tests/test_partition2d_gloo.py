"""World-size-4 runs of the 2-D pr x pc grid orchestration on CPU (gloo),
SURVEY.md §8 f3: GridPxQ slicing, the cfg[0] broadcast down grid columns (F)
/ along grid rows (F*), the cfg[4] all-reduce along rows (F) / down columns
(F*). The per-shard compute is injected (the C oracle) so this checks the
host logic that surrounds the GPU kernels; grids 2x2, 1x4 and 4x1."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import ROOT, rel

NM, ND, NT = 13, 6, 16
GRIDS = [(2, 2), (1, 4), (4, 1)]
CFGS = ("ddddd", "dddds", "sdddd", "sddds")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    rng = np.random.default_rng(7)
    return rng.uniform(-1, 1, NM * ND * NT), rng.uniform(-1, 1, NM * NT), rng.uniform(-1, 1, ND * NT)


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2508_10202_b200 as F
    from oracle.oracle import orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = orc()
        col, m, d = _inputs()
        dims = F.ProblemDims(NM, ND, NT)
        res = {}
        for pr, pc in GRIDS:
            grid = F.GridPxQ.split(pr, pc, ND, NM)
            ri, cj = grid.coords(rank)
            (dlo, dhi), (mlo, mhi) = grid.row_ranges[ri], grid.col_ranges[cj]
            shard = F.shard_operator_2d(F.BlockColumn(dims, col), grid)[rank]
            sop = O.setup_operator(mhi - mlo, dhi - dlo, NT, shard.data)
            dm = F.DistributedMatvec2D(dims, pr, pc, rank, transport="torch",
                                       compute=lambda kind, cfg, x: O.matvec(sop, int(kind), cfg, x))
            for cfg in CFGS:
                res[(pr, pc, "F", cfg)] = (dlo, dhi, dm.forward(m[mlo * NT:mhi * NT] if ri == 0 else None, cfg))
                res[(pr, pc, "A", cfg)] = (mlo, mhi, dm.adjoint(d[dlo * NT:dhi * NT] if cj == 0 else None, cfg))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_grid2d_distributed_gloo(orc):
    import paper_2508_10202_b200 as F

    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    col, m, d = _inputs()
    dims = F.ProblemDims(NM, ND, NT)
    serial = orc.setup_operator(NM, ND, NT, col)
    sf, sa = orc.matvec(serial, 0, "ddddd", m), orc.matvec(serial, 1, "ddddd", d)
    for pr, pc in GRIDS:
        grid = F.GridPxQ.split(pr, pc, ND, NM)
        shards = F.shard_operator_2d(F.BlockColumn(dims, col), grid)
        sops = [orc.setup_operator(s.dims.n_m, s.dims.n_d, NT, s.data) for s in shards]
        pop = F.PartitionedOperator2D(dims, grid, [None] * grid.size)
        for cfg in CFGS:
            # in-process simulation with the same shard compute (fixed tree order)
            run = lambda r, k, c, v: orc.matvec(sops[r], int(k), c, v)  # noqa: E731
            wf = F.partition._matvec_2d(pop, m, cfg, True, run).output.data
            wa = F.partition._matvec_2d(pop, d, cfg, False, run).output.data
            got_f, got_a = np.empty(ND * NT), np.empty(NM * NT)
            for rank in range(world):
                lo, hi, v = out[rank][(pr, pc, "F", cfg)]
                if rank % pc == 0:
                    got_f[lo * NT:hi * NT] = v
                else:  # every rank of a grid row holds the same d slice
                    assert np.array_equal(v, out[rank - rank % pc][(pr, pc, "F", cfg)][2])
                lo, hi, v = out[rank][(pr, pc, "A", cfg)]
                if rank < pc:
                    got_a[lo * NT:hi * NT] = v
                else:
                    assert np.array_equal(v, out[rank % pc][(pr, pc, "A", cfg)][2])
            # <= 2 partials per sum: the all-reduce equals the fixed tree bitwise; 4 partials: to rounding
            tol = 0.0 if max(pr, pc) <= 2 else 1e-15 if cfg[4] == "d" else 1e-6
            assert rel(got_f, wf) <= tol and rel(got_a, wa) <= tol, (pr, pc, cfg)
            if cfg == "ddddd":
                assert rel(got_f, sf) <= 1e-12 and rel(got_a, sa) <= 1e-12, (pr, pc)
            else:
                assert 0 < max(rel(got_f, sf), rel(got_a, sa)) <= 1e-4, (pr, pc, cfg)
        if pr == 1:  # the 1 x p partition (partition.hpp): same numbers as the reference's restatement
            for cfg in CFGS:
                want = orc.matvec_partitioned(NM, ND, NT, col, pc, 0, cfg, m)
                got = out[0][(pr, pc, "F", cfg)][2]
                assert rel(got, want) <= (1e-15 if cfg[4] == "d" else 1e-6), cfg
