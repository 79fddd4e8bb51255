"""ncu target (application replay, cache-control none): SBGEMV-N launched either
right after an F-matvec r2c (mode 'f') or back to back with itself (mode 'g'),
so its DRAM read / write bytes show whether it pays for the r2c's dirty lines."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
mode = sys.argv[1]
NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0); L = F.lib()
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda(); yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
if mode == "f":
    for _ in range(3):
        _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, b"ddddd", ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
else:
    A = torch.randn(100 * 5000 * 1001 + 8, dtype=torch.complex128, device="cuda")
    x = torch.randn(5000 * 1001 + 8, dtype=torch.complex128, device="cuda"); y = torch.empty(100 * 1001, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        _capi.check(L.fmv_sbgemv(ctx.handle, 0, b"z", 100, 5000, 1001, 100, 500000, ctypes.c_void_p(A.data_ptr()), 5000,
                                 ctypes.c_void_p(x.data_ptr()), 100, ctypes.c_void_p(y.data_ptr()), 0, None))
ctx.synchronize()
print("done")
