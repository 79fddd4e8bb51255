"""Sweep ConjTrans SBGEMV knobs on one shape: python tools/tune_conjtrans.py m n batch dtype"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
m, n, b, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
mode = int(sys.argv[5]) if len(sys.argv) > 5 else 2
tdt, es = {"s": (torch.float32, 4), "d": (torch.float64, 8), "c": (torch.complex64, 8), "z": (torch.complex128, 16)}[dt]
A = torch.randn(m * n * b + 8, dtype=tdt, device="cuda")
xl, yl = (n, m) if mode == 0 else (m, n)
x = torch.randn(xl * b + 8, dtype=tdt, device="cuda"); y = torch.empty(yl * b, dtype=tdt, device="cuda")
ctx = F.Context(0); L = F.lib(); torch.cuda.synchronize()
gb = b * (m * n + m + n) * es / 1e9
def run():
    _capi.check(L.fmv_sbgemv(ctx.handle, mode, dt.encode(), m, n, b, m, m * n, ctypes.c_void_p(A.data_ptr()), xl,
                             ctypes.c_void_p(x.data_ptr()), yl, ctypes.c_void_p(y.data_ptr()), 0, None))
grid = [(st, sb, cps, lpc) for lpc in (0, 32, 64, 128, 256) for st in (2, 3, 4) for sb in (32768, 49152, 65536, 98304) for cps in (1, 2)]
for st, sb, cps, lpc in grid:
    os.environ.update(FMV_SBGEMV_STAGES=str(st), FMV_SBGEMV_STAGE_BYTES=str(sb), FMV_SBGEMV_CTAS_PER_SM=str(cps), FMV_SBGEMV_LPC=str(lpc))
    try:
        run(); run(); ctx.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        s = torch.cuda.ExternalStream(ctx.stream_ptr)
        e0.record(s)
        for _ in range(5): run()
        e1.record(s); e1.synchronize()
        t = e0.elapsed_time(e1) / 5
        print(f"lpc={lpc:3d} stages={st} bytes={sb:6d} ctas/sm={cps}: {gb / t * 1e3:6.0f} GB/s", flush=True)
    except Exception as ex:
        print(f"lpc={lpc:3d} stages={st} bytes={sb:6d} ctas/sm={cps}: fail {str(ex)[:60]}", flush=True)
