"""Block (multi-RHS) matvec throughput at C2: K right-hand sides per call,
device-resident I/O, CUDA events on the library stream; prints per-RHS
matvecs/s and the SBGEMV operator-stream GB/s (operator bytes / kernel time)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ddddd"]
Ks = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8, 16]
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
L = F.lib()
res = []
for cfg in cfgs:
    es = {"d": 16, "s": 8}[cfg[2]]
    opb = (NT + 1) * ND * NM * es
    for K in Ks:
        m = torch.from_numpy(F.uniform_fill(K * NM * NT, 2)).cuda()
        d = torch.from_numpy(F.uniform_fill(K * ND * NT, 3)).cuda()
        yo = torch.empty(K * ND * NT, dtype=torch.float64, device="cuda")
        mo = torch.empty(K * NM * NT, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        out = {}
        for kind, x, y in ((0, m, yo), (1, d, mo)):
            call = lambda: _capi.check(L.fmv_matvec_block_async(ctx.handle, op.handle, kind, cfg.encode(), K,
                                                                 ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
            for _ in range(3):
                call()
            ctx.synchronize(); ctx.set_profiling(True); ctx.profile_read(True)
            reps = 6
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            st = torch.cuda.ExternalStream(ctx.stream_ptr)
            s.record(st)
            for _ in range(reps):
                call()
            e.record(st)
            e.synchronize()
            ms, n = ctx.profile_read(True); ctx.set_profiling(False)
            tot = s.elapsed_time(e) / reps
            cls = 1 if kind == 0 else 2
            g_ms = ms[cls] / reps
            out["F" if kind == 0 else "Fstar"] = {"ms_per_call": tot, "rhs_per_s": K / (tot * 1e-3),
                                                  "sbgemv_ms": g_ms, "op_stream_gbs": opb * ((K + 7) // 8) / (g_ms * 1e6)}
        r = {"cfg": cfg, "K": K, **out}
        res.append(r)
        print(json.dumps(r), flush=True)
