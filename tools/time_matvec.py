"""Device-resident F / F* matvec times at C2 (CUDA events on the library's
stream), for A/B runs of environment switches:

  FMV_DEV_CHUNKS=3 python tools/time_matvec.py [--cfg ddddd] [--reps 20]

Prints one JSON line: ms per F, per F*, per step, and the per-kernel-class
times of the step."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="ddddd")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--nm", type=int, default=5000)
ap.add_argument("--nd", type=int, default=100)
ap.add_argument("--nt", type=int, default=1000)
a = ap.parse_args()
NM, ND, NT = a.nm, a.nd, a.nt
col = F.uniform_fill(NM * ND * NT, F.seed_stream(20250814, 0))
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), col), ctx)
del col
m = torch.from_numpy(F.uniform_fill(NM * NT, 1)).cuda()
d = torch.from_numpy(F.uniform_fill(ND * NT, 2)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
L = F.lib()
cb = a.cfg.encode()
st = torch.cuda.ExternalStream(ctx.stream_ptr)


def fwd():
    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, cb, ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))


def adj():
    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, cb, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(mo.data_ptr())))


def timed(fn):
    for _ in range(3):
        fn()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / a.reps


tf, ta = timed(fwd), timed(adj)
ts = timed(lambda: (fwd(), adj()))
ctx.set_profiling(True)
ctx.profile_read(reset=True)
for _ in range(a.reps):
    fwd()
    adj()
ms, n = ctx.profile_read(reset=True)
# host I/O (pinned buffers, blocking fmv_matvec): wall time per call
import time
mp, dp = m.cpu().pin_memory(), d.cpu().pin_memory()
yp, mpo = torch.empty(ND * NT, dtype=torch.float64).pin_memory(), torch.empty(NM * NT, dtype=torch.float64).pin_memory()


def hf():
    _capi.check(L.fmv_matvec(ctx.handle, op.handle, 0, cb, ctypes.c_void_p(mp.data_ptr()), ctypes.c_void_p(yp.data_ptr()), 0, None))


def ha():
    _capi.check(L.fmv_matvec(ctx.handle, op.handle, 1, cb, ctypes.c_void_p(dp.data_ptr()), ctypes.c_void_p(mpo.data_ptr()), 0, None))


def wall(fn):
    for _ in range(3):
        fn()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        fn()
    return (time.perf_counter() - t0) * 1e3 / a.reps


host = {"ms_F": wall(hf), "ms_Fstar": wall(ha), "ms_step": wall(lambda: (hf(), ha()))}
print(json.dumps({"host_pinned": host}))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("FMV_")}, "cfg": a.cfg, "ms_F": tf, "ms_Fstar": ta,
                  "ms_step": ts, "class_ms_per_step": [x / a.reps for x in ms], "class_launches_per_step": [x / a.reps for x in n]}))
