"""SBGEMV-N time in three contexts: back-to-back GEMV only, inside the F matvec, and interleaved with an
fp64 matmul (does the surrounding compute load -- power / clocks -- slow the memory-bound kernel?)."""
import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import torch
import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi
NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0); L = F.lib()
st = torch.cuda.ExternalStream(ctx.stream_ptr)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
m = torch.from_numpy(F.uniform_fill(NM * NT, 2)).cuda(); yo = torch.empty(ND * NT, dtype=torch.float64, device="cuda")
A = torch.randn(100 * 5000 * 1001 + 8, dtype=torch.complex128, device="cuda")
x = torch.randn(5000 * 1001 + 8, dtype=torch.complex128, device="cuda"); y = torch.empty(100 * 1001, dtype=torch.complex128, device="cuda")
gemv = lambda: _capi.check(L.fmv_sbgemv(ctx.handle, 0, b"z", 100, 5000, 1001, 100, 500000, ctypes.c_void_p(A.data_ptr()), 5000, ctypes.c_void_p(x.data_ptr()), 100, ctypes.c_void_p(y.data_ptr()), 0, None))
fwd = lambda: _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, b"ddddd", ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(yo.data_ptr())))
big = torch.randn(2048, 2048, dtype=torch.float64, device="cuda")
def fp64_burn():
    with torch.cuda.stream(st):
        for _ in range(2): big @ big
dirty = torch.empty(10 * 2 ** 20, dtype=torch.float64, device="cuda")  # 80 MB, like r2c's TOSI output
def l2_dirty():
    with torch.cuda.stream(st):
        dirty.fill_(1.0)
small = torch.empty(2 ** 16, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
def l2_read():  # read 80 MB (clean lines), no writes
    with torch.cuda.stream(st):
        sink.copy_(dirty.sum().reshape(1))
def write8():  # 8 MB write
    with torch.cuda.stream(st):
        dirty[: 2 ** 20].fill_(2.0)
flushbuf = torch.empty(20 * 2 ** 20, dtype=torch.float64, device="cuda")  # 160 MB (> L2), clean reads
def l2_dirty_then_evict():  # 80 MB write, then read 160 MB of other data: the dirty lines leave L2 here
    with torch.cuda.stream(st):
        dirty.fill_(1.0)
        sink.copy_(flushbuf.sum().reshape(1))
def l2_dirty_then_sleep():  # 80 MB write, then ~100 us idle: does L2 write dirty lines back on its own?
    with torch.cuda.stream(st):
        dirty.fill_(1.0)
        torch.cuda._sleep(200000)
def tiny():
    with torch.cuda.stream(st):
        small.fill_(1.0)
for name, seq in (("gemv only", [gemv]), ("F matvec", [fwd]), ("gemv + fp64 matmul", [gemv, fp64_burn]),
                  ("80 MB write + gemv", [l2_dirty, gemv]), ("tiny kernel + gemv", [tiny, gemv]),
                  ("80 MB read + gemv", [l2_read, gemv]), ("8 MB write + gemv", [write8, gemv]),
                  ("80MB write, 160MB read, gemv", [l2_dirty_then_evict, gemv]),
                  ("80MB write, idle, gemv", [l2_dirty_then_sleep, gemv])):
    for _ in range(3):
        for f in seq: f()
    ctx.synchronize(); ctx.set_profiling(True); ctx.profile_read(True)
    for _ in range(10):
        for f in seq: f()
    ms, n = ctx.profile_read(True); ctx.set_profiling(False)
    print(f"{name:20s}: SBGEMV-N {ms[1] / n[1] * 1e3:7.1f} us ({8.0897e9 / (ms[1] / n[1] * 1e-3) / 1e9:.0f} GB/s)", flush=True)
