"""NoTrans SBGEMV GB/s for the same 8 GB operator cut into different bin counts
(how much the per-bin flush / cross-CTA reduction costs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

ctx = F.Context(0)
L = F.lib()
st = torch.cuda.ExternalStream(ctx.stream_ptr)
for m, n, b in ((100, 5000, 1001), (100, 50000, 101), (100, 500000, 10), (100, 500, 10001)):
    A = torch.randn(m * n * b + 8, dtype=torch.complex128, device="cuda")
    x = torch.randn(n * b + 8, dtype=torch.complex128, device="cuda")
    y = torch.empty(m * b, dtype=torch.complex128, device="cuda")
    call = lambda: _capi.check(L.fmv_sbgemv(ctx.handle, 0, b"z", m, n, b, m, m * n, ctypes.c_void_p(A.data_ptr()), n,
                                            ctypes.c_void_p(x.data_ptr()), m, ctypes.c_void_p(y.data_ptr()), 0, None))
    for _ in range(3):
        call()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        call()
    e1.record(st)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    gb = b * (m * n + m + n) * 16
    print(f"m={m} n={n} batch={b}: {t * 1e3:.3f} ms  {gb / t / 1e9:.0f} GB/s", flush=True)
    del A, x, y
    torch.cuda.empty_cache()
