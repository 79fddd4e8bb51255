"""C4: conjugate-transpose SBGEMV microbench (BASELINE.json configs[3]).

Grid m in {10,100,1000} x n in {1e3,1e4,1e5}, batch 100, dtypes s/d/c/z,
A m x n column-major, lda=m, stride_a=m*n, op(A)=A^H (A^T for real), the
rocblas-bench layout of PAPER.md:360-362. Cells above 0.8 x free HBM are
skipped. Each timed iteration is preceded by a 512 MB L2 flush and timed
alone with CUDA events (cold_iters 2, iters 10 as PAPER.md:360). GB/s uses the
reference model batch*(m*n+m+n)*elem/s (gemv.hpp:83-89). cuBLAS
<t>gemvStridedBatched is the comparison column (library kernel, not ours).

  python tools/microbench_c4.py [--out profiles/c4_microbench_r01]
"""
import argparse
import ctypes
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_10202_b200 as F
from paper_2508_10202_b200 import _capi

DT = {"s": (torch.float32, 4), "d": (torch.float64, 8), "c": (torch.complex64, 8), "z": (torch.complex128, 16)}


def load_cublas():
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cublas", "lib", "libcublas.so*"))
    cands += glob.glob("/usr/local/cuda/lib64/libcublas.so*")
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/c4_microbench_r02")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--cold", type=int, default=2)
    ap.add_argument("--ms", default="10,100,1000")
    ap.add_argument("--ns", default="1000,10000,100000")
    ap.add_argument("--dtypes", default="sdcz")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = F.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=dev)
    L = F.lib()
    cb = load_cublas()
    handle = ctypes.c_void_p()
    if cb is not None:
        assert cb.cublasCreate_v2(ctypes.byref(handle)) == 0
        cb.cublasSetStream_v2(handle, ctypes.c_void_p(ctx.stream_ptr))
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    rows = []
    batch = 100
    for dt in a.dtypes:
        tdt, es = DT[dt]
        for m in [int(v) for v in a.ms.split(",")]:
            for n in [int(v) for v in a.ns.split(",")]:
                abytes = m * n * batch * es
                free, _ = torch.cuda.mem_get_info(dev)
                if abytes + 64 * 2 ** 20 > 0.8 * free:
                    rows.append({"dtype": dt, "m": m, "n": n, "skipped": f"A is {abytes / 1e9:.1f} GB > 0.8 x free"})
                    continue
                A = torch.randn(m * n * batch + 8, dtype=tdt, device=dev)
                x = torch.randn(m * batch + 8, dtype=tdt, device=dev)
                y = torch.empty(n * batch, dtype=tdt, device=dev)
                y2 = torch.empty(n * batch, dtype=tdt, device=dev)
                torch.cuda.synchronize()

                def ours():
                    _capi.check(L.fmv_sbgemv(ctx.handle, 2, dt.encode(), m, n, batch, m, m * n,
                                             ctypes.c_void_p(A.data_ptr()), m, ctypes.c_void_p(x.data_ptr()), n,
                                             ctypes.c_void_p(y.data_ptr()), 0, None))

                def cublas():
                    one = {"s": ctypes.c_float(1), "d": ctypes.c_double(1), "c": (ctypes.c_float * 2)(1, 0),
                           "z": (ctypes.c_double * 2)(1, 0)}[dt]
                    zero = {"s": ctypes.c_float(0), "d": ctypes.c_double(0), "c": (ctypes.c_float * 2)(0, 0),
                            "z": (ctypes.c_double * 2)(0, 0)}[dt]
                    fn = getattr(cb, {"s": "cublasSgemvStridedBatched", "d": "cublasDgemvStridedBatched",
                                      "c": "cublasCgemvStridedBatched", "z": "cublasZgemvStridedBatched"}[dt])
                    op = 2 if dt in "cz" else 1
                    rc = fn(handle, op, m, n, ctypes.byref(one), ctypes.c_void_p(A.data_ptr()), m,
                            ctypes.c_longlong(m * n), ctypes.c_void_p(x.data_ptr()), 1, ctypes.c_longlong(m),
                            ctypes.byref(zero), ctypes.c_void_p(y2.data_ptr()), 1, ctypes.c_longlong(n), batch)
                    assert rc == 0, rc

                def timeit(fn):
                    ts = []
                    for i in range(a.cold + a.iters):
                        with torch.cuda.stream(stream):
                            flush.zero_()
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        fn()
                        e1.record(stream)
                        e1.synchronize()
                        if i >= a.cold:
                            ts.append(e0.elapsed_time(e1) * 1e-3)
                    return sum(ts) / len(ts)

                t_ours = timeit(ours)
                used = ctypes.c_int(-1)
                _capi.check(L.fmv_sbgemv(ctx.handle, 2, dt.encode(), m, n, batch, m, m * n,
                                         ctypes.c_void_p(A.data_ptr()), m, ctypes.c_void_p(x.data_ptr()), n,
                                         ctypes.c_void_p(y.data_ptr()), 0, ctypes.byref(used)))
                row = {"dtype": dt, "m": m, "n": n, "batch": batch, "ours_s": t_ours,
                       "ours_gbs": F.effective_bandwidth(m, n, batch, es, t_ours), "kernel": {0: "staged", 1: "simple", 2: "small"}[used.value]}
                if cb is not None:
                    t_cb = timeit(cublas)
                    ctx.synchronize()
                    diff = float((y - y2).abs().max() / y2.abs().max())
                    row.update({"cublas_s": t_cb, "cublas_gbs": F.effective_bandwidth(m, n, batch, es, t_cb),
                                "max_rel_diff_vs_cublas": diff})
                row["frac_of_peak"] = row["ours_gbs"] / peak
                rows.append(row)
                print(row, flush=True)
                del A, x, y, y2
                torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump({"peak_gbs": peak, "rows": rows}, open(a.out + ".json", "w"), indent=1)
    md = ["# C4 ConjTrans SBGEMV microbench on 1 x B200", "",
          f"batch 100, lda=m, stride_a=m*n, L2 flushed before each timed call, {a.cold} cold + {a.iters} timed "
          f"iterations; GB/s = batch*(m*n+m+n)*elem/s (gemv.hpp:83-89); peak {peak} GB/s (measured).", "",
          "| dtype | m | n | ours GB/s | frac peak | cuBLAS GB/s | ours/cuBLAS | max rel diff |", "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        if "skipped" in r:
            md.append(f"| {r['dtype']} | {r['m']} | {r['n']} | skipped: {r['skipped']} | | | | |")
            continue
        cg = r.get("cublas_gbs")
        md.append(f"| {r['dtype']} | {r['m']} | {r['n']} | {r['ours_gbs']:.0f} | {r['frac_of_peak']:.2f} | "
                  f"{cg:.0f} | {r['ours_gbs'] / cg:.2f} | {r['max_rel_diff_vs_cublas']:.1e} |" if cg else
                  f"| {r['dtype']} | {r['m']} | {r['n']} | {r['ours_gbs']:.0f} | {r['frac_of_peak']:.2f} | - | - | - |")
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
