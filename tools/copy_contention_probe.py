import ctypes, os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
L = F.lib()
m = torch.from_numpy(F.uniform_fill(NM * NT, 1)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
hp = torch.empty(NM * NT, dtype=torch.float64).pin_memory()
dv = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
cs = torch.cuda.Stream()
st = torch.cuda.ExternalStream(ctx.stream_ptr)
def fwd():
    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, b"ddddd", ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
res = {}
# the device F alone and with a concurrent 40 MB H2D / D2H on another stream
for mode in ("F_alone", "F_with_h2d", "F_with_d2h"):
    ts = []
    for rep in range(8):
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        fwd()
        a1.record(st)
        if mode != "F_alone":
            with torch.cuda.stream(cs):
                if mode == "F_with_h2d":
                    dv.copy_(hp, non_blocking=True)
                else:
                    hp.copy_(dv, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(a0.elapsed_time(a1))
    ts = sorted(ts[2:])
    res[mode] = {"ms": ts[len(ts)//2]}
for mode in ("alone", "with_sbgemv", "d2h_alone", "d2h_with_sbgemv"):
    ts = []
    for rep in range(8):
        torch.cuda.synchronize()
        if "with" in mode:
            fwd()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            e0.record(cs)
            if mode.startswith("d2h"):
                hp.copy_(dv, non_blocking=True)
            else:
                dv.copy_(hp, non_blocking=True)
            e1.record(cs)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    res[mode] = {"ms": ts[len(ts)//2], "GBps": NM * NT * 8 / (ts[len(ts)//2] * 1e6)}
print(json.dumps(res))
