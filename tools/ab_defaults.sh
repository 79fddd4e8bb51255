#!/bin/bash
# SBGEMV kernel GB/s at C2 with the library's default staging, per precision.
for cfg in ddddd dssdd ddhdd; do
  FMV_SBGEMV_STAGES= FMV_SBGEMV_STAGE_BYTES= FMV_SBGEMV_CTAS_PER_SM= timeout 120 python - "$cfg" <<'PY'
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
cfg = sys.argv[1]
NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
op.ensure_single(); op.ensure_half()
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda(); d = torch.from_numpy(F.uniform_fill(ND * NT, 3)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda"); mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
L = F.lib(); es = {"d": 16, "s": 8, "h": 4}[cfg[2]]; gb = (NT + 1) * (ND * NM + ND + NM) * es
res = []
for kind, x, y in ((0, m, yo), (1, d, mo)):
    for _ in range(2):
        _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
    ctx.synchronize(); ctx.set_profiling(True); ctx.profile_read(True)
    for _ in range(10):
        _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
    ms, n = ctx.profile_read(True); ctx.set_profiling(False)
    cls = 1 if kind == 0 else 2
    res.append(gb / (ms[cls] / n[cls]) / 1e6)
print(f"{cfg} defaults: N {res[0]:6.0f} GB/s  C {res[1]:6.0f} GB/s", flush=True)
PY
done
