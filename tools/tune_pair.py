"""A/B of the big Nt=1000 FFT kernels at C2 (FMV_FFT_BIG): persistent prefetching
(fmv_fft_stream.cuh, "stream"), paired-butterfly (fmv_fft_pair.cuh, "pair") and
one-shot one-butterfly-per-thread (k_r2c_reg / k_c2r_reg, "reg"). Prints
per-kernel event times, GB/s against the 120.08 MB algorithmic bytes, and the
relative difference of each output to the "reg" one.

    python tools/tune_pair.py [ddddd,dssdd,...]      (FMV_LIB_PATH=... for a build variant)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda()
d = torch.from_numpy(F.uniform_fill(ND * NT, 3)).cuda()
yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
mo = torch.empty(NM * NT, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
L = F.lib()


def call(kind, cfg):
    x, y = (m, yo) if kind == 0 else (d, mo)
    _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, cfg.encode(), ctypes.c_void_p(x.data_ptr()),
                                   ctypes.c_void_p(y.data_ptr())))


for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["ddddd", "dssdd", "sssss"]):
    outs = {}
    for pair in (os.environ.get("KINDS", "reg,pair,stream").split(",")):
        os.environ["FMV_FFT_BIG"] = pair
        for _ in range(3):
            call(0, cfg)
            call(1, cfg)
        ctx.synchronize()
        outs[pair] = (yo.cpu().numpy().copy(), mo.cpu().numpy().copy())
        ctx.set_profiling(True)
        ctx.profile_read(True)
        for _ in range(20):
            call(0, cfg)
        f_ms, f_n = ctx.profile_read(True)
        for _ in range(20):
            call(1, cfg)
        a_ms, a_n = ctx.profile_read(True)
        ctx.set_profiling(False)
        r2c = f_ms[0] / f_n[0]
        c2r = a_ms[3] / a_n[3]
        print(f"{cfg} {pair:6s}: F r2c {r2c * 1e3:6.1f} us ({120.08e6 / r2c / 1e6:5.0f} GB/s)  "
              f"F* c2r {c2r * 1e3:6.1f} us ({120.08e6 / c2r / 1e6:5.0f} GB/s)  F {sum(f_ms) / 20:.4f} ms  "
              f"F* {sum(a_ms) / 20:.4f} ms", flush=True)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    for k in [x for x in outs if x != "reg"]:
        print(f"{cfg} {k} vs reg: F {rel(outs[k][0], outs['reg'][0]):.2e}  F* {rel(outs[k][1], outs['reg'][1]):.2e}",
              flush=True)
