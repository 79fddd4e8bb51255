"""Host-I/O matvec times at C2 through fmv_matvec: pinned vs pageable input and
output buffers, per FMV_CHUNKS (the reference-API drop-in path passes
pageable std::vectors). Prints one JSON line per (chunks, kind, in, out).

    FMV_HOST_THREADS=8 python tools/pageable_probe.py [chunks,...]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

NM, ND, NT = 5000, 100, 1000
ctx = F.Context(0)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), F.uniform_fill(NM * ND * NT, 1)), ctx)
L = F.lib()
bufs = {}
for name, n in (("m", NM * NT), ("d", ND * NT)):
    a = F.uniform_fill(n, 7)
    bufs[(name, "pageable")] = a.copy()
    t = torch.empty(n, dtype=torch.float64).pin_memory()
    t.numpy()[:] = a
    bufs[(name, "pinned")] = t.numpy()
    bufs[(name + "_out", "pageable")] = np.zeros(n)
    bufs[(name + "_out", "pinned")] = torch.zeros(n, dtype=torch.float64).pin_memory().numpy()


def call(kind, x, y):
    _capi.check(L.fmv_matvec(ctx.handle, op.handle, kind, b"ddddd", x.ctypes.data_as(ctypes.c_void_p),
                             y.ctypes.data_as(ctypes.c_void_p), 0, None))


for chunks in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "3", "6", "12"]):
    os.environ["FMV_CHUNKS"] = chunks
    for kind in (0, 1):
        xin, xout = ("m", "d_out") if kind == 0 else ("d", "m_out")
        for ik in ("pinned", "pageable"):
            for ok in ("pinned", "pageable"):
                x, y = bufs[(xin, ik)], bufs[(xout, ok)]
                for _ in range(3):
                    call(kind, x, y)
                R = 10
                t0 = time.perf_counter()
                for _ in range(R):
                    call(kind, x, y)
                ms = (time.perf_counter() - t0) / R * 1e3
                print(json.dumps({"chunks": chunks, "kind": "F" if kind == 0 else "F*", "in": ik, "out": ok,
                                  "ms": round(ms, 4), "host_threads": os.environ.get("FMV_HOST_THREADS", "")}),
                      flush=True)
