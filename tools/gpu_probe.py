"""Developer probe: parity + timing of the B200 path against the reference oracle."""
import os, sys, time
os.environ.setdefault("MKL_NUM_THREADS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_10202_b200 as F
from oracle.oracle import ref

R = ref()
S = 20250814


def case(nm, nd, nt, cfgs=("ddddd",), fill="uni", dense=True):
    if fill == "uni":
        col = F.uniform_fill(nm * nd * nt, F.seed_stream(S, 0))
        m = F.uniform_fill(nm * nt, F.seed_stream(S, 1))
        d = F.uniform_fill(nd * nt, F.seed_stream(S, 2))
    else:
        col = F.non_representable_fill(nm * nd * nt, F.seed_stream(S, 0))
        m = F.non_representable_fill(nm * nt, F.seed_stream(S, 1))
        d = F.non_representable_fill(nd * nt, F.seed_stream(S, 2))
    t0 = time.time()
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    tg = time.time() - t0
    t0 = time.time()
    rop = R.setup_operator(nm, nd, nt, col)
    tr = time.time() - t0
    bg = op.bins_double
    br = rop.bins()
    eb = np.linalg.norm(bg - br) / np.linalg.norm(br)
    print(f"[{nm},{nd},{nt}] setup gpu {tg:.3f}s ref {tr:.3f}s bins rel {eb:.3e}", flush=True)
    r0f = R.matvec(rop, 0, "ddddd", m)
    r0a = R.matvec(rop, 1, "ddddd", d)
    for cfg in cfgs:
        rf = R.matvec(rop, 0, cfg, m) if "h" not in cfg else r0f
        ra = R.matvec(rop, 1, cfg, d) if "h" not in cfg else r0a
        gf = F.forward_matvec(op, m, cfg).output.data
        ga = F.adjoint_matvec(op, d, cfg).output.data
        ef = np.linalg.norm(gf - rf) / np.linalg.norm(rf)
        ea = np.linalg.norm(ga - ra) / np.linalg.norm(ra)
        erf = np.linalg.norm(rf - r0f) / np.linalg.norm(r0f)
        egf = np.linalg.norm(gf - r0f) / np.linalg.norm(r0f)
        era = np.linalg.norm(ra - r0a) / np.linalg.norm(r0a)
        ega = np.linalg.norm(ga - r0a) / np.linalg.norm(r0a)
        print(f"  {cfg}: F gpu-vs-ref {ef:.3e} (err vs ddddd: ref {erf:.3e} gpu {egf:.3e}) | "
              f"F* gpu-vs-ref {ea:.3e} (ref {era:.3e} gpu {ega:.3e})", flush=True)
    if dense and nd * nm * nt * nt <= 1e8:
        df = R.dense(0, nm, nd, nt, col, m)
        da = R.dense(1, nm, nd, nt, col, d)
        gf = F.forward_matvec(op, m).output.data
        ga = F.adjoint_matvec(op, d).output.data
        print(f"  dense: F {np.linalg.norm(gf-df)/np.linalg.norm(df):.3e} F* {np.linalg.norm(ga-da)/np.linalg.norm(da):.3e}")
    return op


def bench(op, nm, nd, nt, cfg="ddddd", iters=20):
    ctx = op.ctx
    dev = torch.device("cuda:0")
    m = torch.randn(nm * nt, dtype=torch.float64, device=dev)
    d = torch.randn(nd * nt, dtype=torch.float64, device=dev)
    dout = torch.empty(nd * nt, dtype=torch.float64, device=dev)
    mout = torch.empty(nm * nt, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    L = F.lib()
    s = torch.cuda.ExternalStream(ctx.stream_ptr)
    for kind, x, y, name in ((0, m, dout, "F"), (1, d, mout, "F*")):
        for _ in range(3):
            F._capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), x.data_ptr(), y.data_ptr()))
        ctx.synchronize()
        ctx.set_profiling(True)
        ctx.profile_read(True)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(iters):
            F._capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), x.data_ptr(), y.data_ptr()))
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / iters
        kms, kn = ctx.profile_read(True)
        ctx.set_profiling(False)
        nb = nt + 1
        es = {"d": 16, "s": 8, "h": 4}[cfg[2]]
        gb = nb * (nd * nm + nd + nm) * es / 1e9
        gk = kms[1 if kind == 0 else 2] / max(1, kn[1 if kind == 0 else 2])
        print(f"  {name} {cfg}: {ms:.3f} ms/matvec ({1000/ms:.1f}/s); kernels ms: r2c {kms[0]/iters:.3f} "
              f"gemv {gk:.3f} ({gb/gk*1e3:.0f} GB/s) c2r {kms[3]/iters:.3f}", flush=True)


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0), flush=True)
    case(100, 10, 100, cfgs=("ddddd", "dssdd", "sssss", "ddsdd", "dddds", "ddsss", "ddhdd", "hdhdh"))
    case(16, 8, 32, dense=True)
    case(5, 3, 8, cfgs=("ddddd", "sssss"))
    case(7, 3, 1)
    case(13, 5, 7, cfgs=("ddddd", "dssdd"))
    case(17, 3, 11)
    case(64, 4, 32)
    case(500, 20, 200, cfgs=("ddddd", "dssdd", "ddsdd", "ddhdd"), fill="nonrep")
    op = case(5000, 100, 1000, cfgs=("ddddd", "dssdd"), dense=False)
    bench(op, 5000, 100, 1000, "ddddd")
    bench(op, 5000, 100, 1000, "dssdd")
    bench(op, 5000, 100, 1000, "ddhdd")
