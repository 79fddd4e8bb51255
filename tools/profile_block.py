"""ncu target: block (multi-RHS) matvecs at C2 -- F with K = 8 and F* with K = 4, after one warm-up each."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
L = F.lib()
for kind, K, n_in, n_out in ((0, 8, NM, ND), (1, 4, ND, NM)):
    X = torch.from_numpy(F.uniform_fill(K * n_in * NT, 2)).cuda()
    Y = torch.empty(K * n_out * NT, dtype=torch.float64, device="cuda")
    for _ in range(2):
        _capi.check(L.fmv_matvec_block_async(ctx.handle, op.handle, kind, b"ddddd", K, ctypes.c_void_p(X.data_ptr()),
                                             ctypes.c_void_p(Y.data_ptr())))
ctx.synchronize()
print("done")
