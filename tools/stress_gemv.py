"""Bitwise stress: staged SBGEMV repeated many times vs the first result (races show up as flips)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_10202_b200 as F
m, n, b, mode, dt, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], int(sys.argv[6])
tdt = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}[dt]
A = torch.randn(m * n * b + 8, dtype=tdt, device="cuda"); xl = n if mode == 0 else m
x = torch.randn(xl * b + 8, dtype=tdt, device="cuda"); yl = m if mode == 0 else n
y0 = torch.empty(yl * b, dtype=tdt, device="cuda"); y = torch.empty_like(y0)
F.gemv_batched(F.GemvMode(mode), dt, m, n, b, m, m * n, A, xl, x, yl, y0)
ys, _ = F.gemv_batched(F.GemvMode(mode), dt, m, n, b, m, m * n, A, xl, x, yl, torch.empty_like(y0), force_simple=True)
bad = 0
for i in range(reps):
    F.gemv_batched(F.GemvMode(mode), dt, m, n, b, m, m * n, A, xl, x, yl, y)
    bad += int(not torch.equal(y, y0))
err = float((y0 - ys).abs().max() / ys.abs().max())
print(f"m={m} n={n} b={b} mode={mode} {dt}: {bad}/{reps} runs differ bitwise; max rel diff vs simple {err:.2e}")
