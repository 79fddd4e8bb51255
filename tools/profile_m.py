"""ncu target: F* SBGEMV at C2 for the 's' and 'm' SBGEMV precisions (ddsdd, ddmdd), one call each after a warm-up."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
L = F.lib()
d = torch.from_numpy(F.uniform_fill(ND * NT, 2)).cuda()
mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
for cfg in (b"ddsdd", b"ddmdd"):
    for _ in range(2):
        _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, cfg, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(mo.data_ptr())))
ctx.synchronize()
print("done")
