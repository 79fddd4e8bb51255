"""Sweep the SBGEMV staging knobs (ring depth, stage bytes, CTAs/SM) at C2 and print kernel GB/s."""
import ctypes, itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ddddd", "dssdd", "ddhdd"]
col = F.uniform_fill(NM * ND * NT, 1)
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), col), ctx)
op.ensure_single(); op.ensure_half()
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda(); d = torch.from_numpy(F.uniform_fill(ND * NT, 3)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda"); mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
L = F.lib()
nb = NT + 1
grid = [(st, sb, cps) for st in (3, 4, 6, 8) for sb in (16384, 24576, 32768, 49152) for cps in (1, 2)]
if len(sys.argv) > 2 and sys.argv[2] == "env":  # one row from the caller's FMV_SBGEMV_* environment
    grid = [(int(os.environ.get("FMV_SBGEMV_STAGES", 3)), int(os.environ.get("FMV_SBGEMV_STAGE_BYTES", 32768)),
             int(os.environ.get("FMV_SBGEMV_CTAS_PER_SM", 2)))]
elif len(sys.argv) > 2 and sys.argv[2] == "quick":
    grid = [(4, 24576, 2), (6, 16384, 2), (8, 12288, 2), (3, 32768, 2), (8, 24576, 1)]
for cfg in cfgs:
    es = {"d": 16, "s": 8, "h": 4}[cfg[2]]
    gb = nb * (ND * NM + ND + NM) * es
    for st, sb, cps in grid:
        if st * sb > 200 * 1024 * (2 if cps == 1 else 1) / 1:
            pass
        os.environ["FMV_SBGEMV_STAGES"] = str(st)
        os.environ["FMV_SBGEMV_STAGE_BYTES"] = str(sb)
        os.environ["FMV_SBGEMV_CTAS_PER_SM"] = str(cps)
        res = []
        for kind, x, y in ((0, m, yo), (1, d, mo)):
            try:
                for _ in range(2):
                    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
                ctx.synchronize(); ctx.set_profiling(True); ctx.profile_read(True)
                for _ in range(8):
                    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
                ms, n = ctx.profile_read(True); ctx.set_profiling(False)
                cls = 1 if kind == 0 else 2
                t = ms[cls] / n[cls]
                res.append(f"{gb / t / 1e6:6.0f}")
            except Exception as e:
                res.append("  fail")
                ctx.set_profiling(False)
        print(f"{cfg} stages={st} bytes={sb:6d} ctas/sm={cps}: N {res[0]} GB/s  C {res[1]} GB/s", flush=True)
