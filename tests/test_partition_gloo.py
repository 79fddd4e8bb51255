"""World-size-2 runs of the distributed partition host logic on CPU (gloo):
Grid1xP slicing, the cfg[0] broadcast payload, the cfg[4] all-reduce and
shard concatenation. The per-shard compute is injected (the C oracle), so
this checks the orchestration that runs around the GPU kernels on B200."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, rel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


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
        nm, nd, nt = 13, 3, 16
        rng = np.random.default_rng(0)
        col = rng.uniform(-1, 1, nm * nd * nt)
        m = rng.uniform(-1, 1, nm * nt)
        d = rng.uniform(-1, 1, nd * nt)
        dims = F.ProblemDims(nm, nd, nt)
        grid = F.Grid1xP.split(world, nm)
        lo, hi = grid.shard_ranges[rank]
        shard = F.shard_operator(F.BlockColumn(dims, col), grid)[rank]
        sop = O.setup_operator(hi - lo, nd, nt, shard.data)
        dm = F.DistributedMatvec(dims, rank, world, transport="torch",
                                 compute=lambda kind, cfg, x: O.matvec(sop, int(kind), cfg, x))
        res = {}
        for cfg in ("ddddd", "dddds", "sdddd", "hdddh"):
            res["F_" + cfg] = dm.forward(m[lo * nt:hi * nt], cfg)
            res["A_" + cfg] = dm.adjoint(d if rank == 0 else None, cfg)
        q.put((rank, lo, hi, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_partition_gloo(world, orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    nm, nd, nt = 13, 3, 16
    rng = np.random.default_rng(0)
    col = rng.uniform(-1, 1, nm * nd * nt)
    m = rng.uniform(-1, 1, nm * nt)
    d = rng.uniform(-1, 1, nd * nt)
    serial = orc.setup_operator(nm, nd, nt, col)
    for cfg in ("ddddd", "dddds", "sdddd"):
        want_f = orc.matvec_partitioned(nm, nd, nt, col, world, 0, cfg, m)
        want_a = orc.matvec_partitioned(nm, nd, nt, col, world, 1, cfg, d)
        for rank, lo, hi, res in out:
            # all-reduce vs the reference's fixed tree: identical for p=2 (one addition)
            assert rel(res["F_" + cfg], want_f) < 1e-15
            assert np.array_equal(res["A_" + cfg], want_a[lo * nt:hi * nt])  # broadcast + shard: bitwise
        if cfg == "ddddd":
            assert rel(out[0][3]["F_ddddd"], orc.matvec(serial, 0, "ddddd", m)) < 1e-12
    e = rel(out[0][3]["F_dddds"], orc.matvec(serial, 0, "ddddd", m))
    assert 0 < e <= 1e-4
    eh = rel(out[0][3]["F_hdddh"], orc.matvec(serial, 0, "ddddd", m))
    assert 0 < eh <= 5e-3
