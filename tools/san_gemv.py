"""Isolated SBGEMV shapes for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_10202_b200 as F
m, n, b, mode, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
rng = np.random.default_rng(0)
npdt = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}[dt]
A = rng.standard_normal(m * n * b).astype(npdt)
xl = n if mode == 0 else m
x = rng.standard_normal(xl * b).astype(npdt)
y, used = F.gemv_batched(F.GemvMode(mode), dt, m, n, b, m, m * n, A, xl, x, n if mode else m)
print("ok", used, float(np.abs(y).sum()))
