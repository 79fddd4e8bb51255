"""e2e (host-buffer) matvec time at C2 vs the column-chunk count of the
host-I/O pipeline (FMV_CHUNKS), F and F* separately, pinned host buffers."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
L = F.lib()
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).pin_memory()
d = torch.from_numpy(F.uniform_fill(ND * NT, 3)).pin_memory()
do = torch.empty(ND * NT, dtype=torch.float64).pin_memory()
mo = torch.empty(NM * NT, dtype=torch.float64).pin_memory()
cfg = (sys.argv[1] if len(sys.argv) > 1 else "ddddd").encode()
for ch in [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "1,3,6,8,12,16").split(",")]:
    os.environ["FMV_CHUNKS"] = str(ch)
    res = []
    for kind, x, y in ((0, m, do), (1, d, mo)):
        call = lambda: _capi.check(L.fmv_matvec(ctx.handle, op.handle, kind, cfg, ctypes.c_void_p(x.data_ptr()),
                                                 ctypes.c_void_p(y.data_ptr()), 0, None))
        for _ in range(3):
            call()
        t0 = time.perf_counter()
        for _ in range(10):
            call()
        res.append((time.perf_counter() - t0) / 10 * 1e3)
    print(f"chunks={ch:2d}: F {res[0]:.3f} ms  F* {res[1]:.3f} ms  step {res[0] + res[1]:.3f} ms", flush=True)
