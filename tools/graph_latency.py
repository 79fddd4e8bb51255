"""Per-matvec latency at C1 (Nm=100, Nd=10, Nt=100) and C2: direct device-resident
calls (fmv_matvec_async) vs CUDA-graph replays (fmv_graph_launch), 200 back-to-back
calls timed with CUDA events on the context stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

for nm, nd, nt, reps in ((100, 10, 100, 200), (5000, 100, 1000, 20)):
    ctx = F.Context(0)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), F.uniform_fill(nm * nd * nt, 1)), ctx)
    st = torch.cuda.ExternalStream(ctx.stream_ptr)
    L = F.lib()
    for kind, n_in, n_out in ((0, nm * nt, nd * nt), (1, nd * nt, nm * nt)):
        x = torch.from_numpy(F.uniform_fill(n_in, 2)).cuda()
        y = torch.empty(n_out, dtype=torch.float64, device="cuda")
        direct = lambda: _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, b"ddddd", ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
        g = F.MatvecGraph(op, F.MatvecKind(kind), x, y, "ddddd", ctx)
        res = {}
        for name, fn in (("direct", direct), ("graph", g.launch)):
            for _ in range(5):
                fn()
            ctx.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                fn()
            e1.record(st)
            e1.synchronize()
            res[name] = e0.elapsed_time(e1) / reps * 1e3
        print(f"{nm}/{nd}/{nt} {'F ' if kind == 0 else 'F*'}: direct {res['direct']:8.1f} us  graph {res['graph']:8.1f} us", flush=True)
        del g
