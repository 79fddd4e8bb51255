"""ncu target: C2 operator, 2 warm-up steps then 2 profiled steps (F + F*)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

cfg = (sys.argv[1] if len(sys.argv) > 1 else "ddddd").encode()
NM, ND, NT = 5000, 100, 1000
col = F.uniform_fill(NM * ND * NT, F.seed_stream(20250814, 0))
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), col), ctx)
m = torch.from_numpy(F.uniform_fill(NM * NT, 1)).cuda()
d = torch.from_numpy(F.uniform_fill(ND * NT, 2)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
L = F.lib()
for _ in range(4):
    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, cfg, ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, cfg, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(mo.data_ptr())))
ctx.synchronize()
print("done")
