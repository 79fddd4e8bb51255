"""Big-FFT phase GB/s at time lengths other than the two specialised ones:
F's r2c over Nm series and F*'s c2r over Nm series inside device-resident
matvecs (CUDA events per kernel class), Nm*Nt ~ 5e6 samples as at C2.
Algorithmic bytes per transform: Nm*Nt*8 (real side) + Nm*(Nt+1)*16 (bins).

    python tools/fft_lengths_bench.py [nt,...]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

ND = 4
L = F.lib()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6548.0
for nt in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else "512,1000,1024,2000,4096,8192".split(","))]:
    nm = max(1024, 5_000_000 // nt)
    ctx = F.Context(0)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, ND, nt), F.uniform_fill(nm * ND * nt, 1)), ctx)
    m = torch.from_numpy(F.uniform_fill(nm * nt, 2)).cuda()
    d = torch.from_numpy(F.uniform_fill(ND * nt, 3)).cuda()
    yo = torch.empty(ND * nt, dtype=torch.float64, device="cuda")
    mo = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()

    def call(kind):
        x, y = (m, yo) if kind == 0 else (d, mo)
        _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, kind, b"ddddd", ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr())))

    for _ in range(3):
        call(0)
        call(1)
    ctx.synchronize()
    ctx.set_profiling(True)
    ctx.profile_read(True)
    R = 10
    for _ in range(R):
        call(0)
    f_ms, f_n = ctx.profile_read(True)
    for _ in range(R):
        call(1)
    a_ms, a_n = ctx.profile_read(True)
    ctx.set_profiling(False)
    byts = nm * nt * 8 + nm * (nt + 1) * 16
    r2c = f_ms[0] / R  # F: one big r2c (Nm series) per matvec
    c2r = a_ms[3] / R  # F*: one big c2r (Nm series) per matvec
    print(json.dumps({"nt": nt, "nm": nm, "r2c_us": round(r2c * 1e3, 1), "r2c_gbs": round(byts / r2c / 1e6),
                      "c2r_us": round(c2r * 1e3, 1), "c2r_gbs": round(byts / c2r / 1e6),
                      "frac_of_peak": round(2 * byts / (r2c + c2r) / 1e6 / peak, 3),
                      "launches_r2c": f_n[0] / R, "launches_c2r": a_n[3] / R}), flush=True)
    del op, ctx
