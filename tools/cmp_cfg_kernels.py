"""Per-kernel-class times of F at C2 for a few precision configs (device I/O)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
op.ensure_single(); op.ensure_half()
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda(); yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
L = F.lib()
st = torch.cuda.ExternalStream(ctx.stream_ptr)
for cfg in ("ddhdd", "ddhsd", "ddsdd", "ddssd", "ddddd"):
    call = lambda: _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, cfg.encode(), ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
    for _ in range(3): call()
    ctx.synchronize(); ctx.set_profiling(True); ctx.profile_read(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10): call()
    e1.record(st); e1.synchronize()
    ms, n = ctx.profile_read(True); ctx.set_profiling(False)
    print(cfg, "total %.3f ms" % (e0.elapsed_time(e1) / 10), " per-class ms:", [round(ms[i] / 10, 4) for i in range(5)], [int(n[i]) for i in range(5)])
