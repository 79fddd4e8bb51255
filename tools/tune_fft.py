"""Time the big-FFT kernels (F r2c over Nm series, F* c2r over Nm series) at C2: register-resident
radix-10 kernels vs the general mixed-radix (legacy) kernels."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda(); d = torch.from_numpy(F.uniform_fill(ND * NT, 3)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda"); mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); L = F.lib()
for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["ddddd", "dssdd"]):
    for legacy in (1, 0):
        os.environ["FMV_FFT_LEGACY"] = str(legacy)
        for _ in range(2):
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, cfg.encode(), ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, cfg.encode(), ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(mo.data_ptr())))
        ctx.synchronize(); ctx.set_profiling(True); ctx.profile_read(True)
        for _ in range(10):
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, cfg.encode(), ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
        f_ms, f_n = ctx.profile_read(True)
        for _ in range(10):
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, cfg.encode(), ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(mo.data_ptr())))
        a_ms, a_n = ctx.profile_read(True); ctx.set_profiling(False)
        r2c = f_ms[0] / f_n[0]; c2r = a_ms[3] / a_n[3]
        print(f"{cfg} {'legacy' if legacy else 'reg   '}: F r2c {r2c*1e3:7.1f} us ({120.08e6/r2c/1e6:6.0f} GB/s)  F* c2r {c2r*1e3:7.1f} us ({120.08e6/c2r/1e6:6.0f} GB/s)  small r2c {a_ms[0]/a_n[0]*1e3:5.1f} us small c2r {f_ms[3]/f_n[3]*1e3:5.1f} us", flush=True)
