#!/usr/bin/env python
"""Benchmark of the B200 FFTMatvec hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--cfg ddddd]

One STEP = one forward (d = F m) + one adjoint (m = F* d) matvec on the C2
operator (Nm=5000, Nd=100, Nt=1000; 8.0 GB of complex128 bins per GPU), so
the unit of work is one "shard-matvec" over an Nm=5000 column block. At N
GPUs (torchrun, one rank per GPU) each rank holds its own Nm=5000 shard of an
Nm=5000*N operator (weak scaling, partition.hpp 1 x p grid): one distributed
F is N shard-matvecs + an NCCL all-gather of the partial d summed by a fixed tree, one distributed F* is an NCCL
broadcast of d + N shard-matvecs.

value   : shard-matvecs/s of the whole job, device-resident inputs (HBM).
e2e     : the same through the C ABI with pinned HOST buffers (H2D of every
          step's inputs and D2H of its outputs inside the timed region):
          queued calls (fmv_matvec_host_async; each call's copies overlap
          its neighbours' compute) at N=1, blocking fmv_matvec /
          fmv_matvec_partitioned otherwise; e2e_blocking: the blocking call.
roofline: SBGEMV kernels (the dominant phase, ~90% of a matvec) -- reference
          algorithmic bytes nb*(Nd*Nm+Nd+Nm)*16 per launch (gemv.hpp:83-89,
          SURVEY.md §8d) / CUDA-event kernel time, vs MEASURED_PEAKS.json.
cpu_baseline / --impl reference: the reference itself (oracle/_ref: the
          reference headers compiled verbatim) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("MKL_NUM_THREADS", "1")
# NCCL prints its version banner on stdout at init; keep stdout for the one JSON line
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
if int(os.environ.get("WORLD_SIZE", "1")) > 1:
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator size / transport in the driver's stderr log
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import ctypes  # noqa: E402

import numpy as np  # noqa: E402

SEED = 20250814
NM, ND, NT = 5000, 100, 1000  # C2 (BASELINE.json configs[1]); --workload c5 switches to Nd=600 (configs[4])
METRIC = "F and F* matvecs/sec at 1/2/4/8 B200; SBGEMV+FFT HBM GB/s vs peak"
UNIT = "matvecs/s"


def env_int(name, dflt):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else dflt


def measured_peak_gbs():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch DRAM bytes of the SBGEMV kernels from the committed ncu capture."""
    p = os.path.join(HERE, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling of SM clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm_, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm_)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(rank: int):
    """Synthetic inputs from the reference generators (random_fill.hpp), seeded per shard."""
    import paper_2508_10202_b200 as F

    base = F.seed_stream(SEED, 1000 + rank) if rank else SEED
    col = F.uniform_fill(NT * ND * NM, F.seed_stream(base, 0))
    m = F.uniform_fill(NM * NT, F.seed_stream(base, 1))
    d = F.uniform_fill(ND * NT, F.seed_stream(SEED, 2))  # d is global (broadcast from rank 0)
    return col, m, d


# ------------------------------------------------------------- reference ---
def ref_setup(col):
    from oracle.oracle import ref

    R = ref()
    t0 = time.time()
    op = R.setup_operator(NM, ND, NT, col)
    return R, op, time.time() - t0


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_inputs(R):
    """make_inputs() through the reference's own generators (oracle/_ref:
    random_fill.hpp compiled verbatim): the same bits, and nothing of this
    repo's package is loaded in the reference arm."""
    col = R.uniform_fill(NT * ND * NM, R.seed_stream(SEED, 0))
    m = R.uniform_fill(NM * NT, R.seed_stream(SEED, 1))
    d = R.uniform_fill(ND * NT, R.seed_stream(SEED, 2))
    return col, m, d


def run_reference_arm(args, rank, world):
    if rank != 0:
        return None
    from oracle.oracle import ref

    col, m, d = ref_inputs(ref())
    R, op, t_setup = ref_setup(col)
    T = cpu_threads()
    cfg = args.cfg
    for _ in range(args.warmup):
        R.throughput_mixed(op, cfg, m, d, T)
    t = 0.0
    for _ in range(args.steps):
        t += R.throughput_mixed(op, cfg, m, d, T)
    value = args.steps * T / t
    sample = (f"each step: {T} host threads run concurrently on one shared C2 operator, even threads one F, odd "
              f"threads one F* (reference forward_matvec/adjoint_matvec, cfg {cfg}); setup_operator {t_setup:.1f}s "
              f"excluded")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if cfg == "ddddd" else "mixed", "data": "synthetic",
        "config": workload_config(world, cfg),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def workload_config(world, cfg):
    name = "C2" if ND == 100 else "C5"
    return {"workload": f"{name} FFTMatvec Nm={NM}/GPU Nd={ND} Nt={NT}, cfg {cfg}, step = 1 F + 1 F*",
            "n_m_per_gpu": NM, "n_d": ND, "n_t": NT, "n_m_total": NM * world, "precision_config": cfg,
            "operator_bytes_per_gpu": (NT + 1) * ND * NM * 16,
            "l2": f"inputs larger than L2: the {(NT + 1) * ND * NM * 16 / 1e9:.1f} GB operator is streamed once per matvec",
            "parallelism": f"1x{world} column partition" + (" (NCCL all-gather + fixed-tree reduce for F, broadcast for F*)" if world > 1 else ""),
            "matvec_unit": "one F or F* over an Nm=5000 shard; a distributed matvec on N GPUs = N units"}


# ------------------------------------------------------------------- ours ---
def run_ours(args, rank, world, device):
    import torch

    import paper_2508_10202_b200 as F
    from paper_2508_10202_b200 import _capi

    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

    col, m_h, d_h = make_inputs(rank)
    ctx = F.Context(device)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), col), ctx)
    cfg = args.cfg
    if cfg[2] == "s":
        op.ensure_single()
    if cfg[2] == "h":
        op.ensure_half()
    L = F.lib()
    cb = cfg.encode()
    m = torch.from_numpy(m_h).to(dev)
    d = torch.from_numpy(d_h).to(dev)
    dout = torch.empty(ND * NT, dtype=torch.float64, device=dev)
    mout = torch.empty(NM * NT, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=dev)
    dm = None
    if world > 1 or os.environ.get("FMV_BENCH_FORCE_DIST") == "1":  # (the latter: exercise the NCCL path on 1 GPU)
        dm = F.DistributedMatvec(F.ProblemDims(NM * world, ND, NT), rank, world, shard=op, transport="native", ctx=ctx)
        nranks, crank = dm.comm_size()
        if nranks != world or crank != rank:
            raise SystemExit(f"bench: communicator has {nranks} ranks (this rank {crank}), expected {world} ({rank})")

    def step_device():
        if dm is None:
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 0, cb, ctypes.c_void_p(m.data_ptr()),
                                           ctypes.c_void_p(dout.data_ptr())))
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, cb, ctypes.c_void_p(d.data_ptr()),
                                           ctypes.c_void_p(mout.data_ptr())))
        else:  # enqueued like the single-GPU path; ctx.synchronize() waits under the NCCL watch
            for kind, x, y in ((0, m, dout), (1, d, mout)):
                _capi.check(L.fmv_matvec_partitioned_async(ctx.handle, op.handle, kind, cb,
                                                           ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))

    def barrier():
        if dist is not None:
            dist.barrier()

    def timed(fn, k, join=False):
        barrier()
        ctx.synchronize()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        if join:  # the queued calls' output copies run on a side stream
            _capi.check(L.fmv_join(ctx.handle))
        e1.record(stream)
        e1.synchronize()
        ctx.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---- device-resident throughput (value) + per-kernel CUDA events
    clk = ClockSampler(device).__enter__()  # samples through warm-up, timed and e2e regions
    for _ in range(args.warmup):
        step_device()
    ctx.synchronize()
    ctx.set_profiling(True)
    ctx.profile_read(reset=True)
    l0 = ctx.launches()
    ms = timed(step_device, args.steps)
    launches = ctx.launches() - l0
    kms, kn = ctx.profile_read(reset=True)
    ctx.set_profiling(False)
    value = 2 * args.steps * world / (ms * 1e-3)

    # ---- end to end through the C ABI with pinned host buffers (e2e)
    m_pin = torch.from_numpy(m_h).pin_memory()
    d_pin = torch.from_numpy(d_h).pin_memory()
    do_pin = torch.empty(ND * NT, dtype=torch.float64).pin_memory()
    mo_pin = torch.empty(NM * NT, dtype=torch.float64).pin_memory()

    def step_host():
        if dm is None:
            _capi.check(L.fmv_matvec(ctx.handle, op.handle, 0, cb, ctypes.c_void_p(m_pin.data_ptr()),
                                     ctypes.c_void_p(do_pin.data_ptr()), 0, None))
            _capi.check(L.fmv_matvec(ctx.handle, op.handle, 1, cb, ctypes.c_void_p(d_pin.data_ptr()),
                                     ctypes.c_void_p(mo_pin.data_ptr()), 0, None))
        else:
            for kind, x, y in ((0, m_pin, do_pin), (1, d_pin, mo_pin)):
                _capi.check(L.fmv_matvec_partitioned(ctx.handle, op.handle, kind, cb, ctypes.c_void_p(x.data_ptr()),
                                                     ctypes.c_void_p(y.data_ptr()), 0, None))

    def step_host_queued():
        _capi.check(L.fmv_matvec_host_async(ctx.handle, op.handle, 0, cb, ctypes.c_void_p(m_pin.data_ptr()),
                                            ctypes.c_void_p(do_pin.data_ptr())))
        _capi.check(L.fmv_matvec_host_async(ctx.handle, op.handle, 1, cb, ctypes.c_void_p(d_pin.data_ptr()),
                                            ctypes.c_void_p(mo_pin.data_ptr())))

    for _ in range(max(3, args.warmup // 2)):
        step_host()
    ms_blk = timed(step_host, args.steps)
    e2e_api = "fmv_matvec (C ABI, blocking), pinned host buffers"
    ms_e2e = ms_blk
    if dm is None:
        for _ in range(max(3, args.warmup // 2)):
            step_host_queued()
        ctx.synchronize()
        ms_e2e = timed(step_host_queued, args.steps, join=True)
        e2e_api = "fmv_matvec_host_async (C ABI, queued F and F* calls), pinned host buffers"
    clk.__exit__(None, None, None)
    e2e_value = 2 * args.steps * world / (ms_e2e * 1e-3)
    h2d = (NM * NT + ND * NT) * 8 * world
    d2h = (ND * NT + NM * NT) * 8 * world

    # ---- roofline of the dominant kernel (SBGEMV N + C)
    peak, peak_src = measured_peak_gbs()
    es = {"d": 16, "s": 8, "h": 4}[cfg[2]]
    nb = NT + 1
    gemv_bytes = nb * (ND * NM + ND + NM) * es  # gemv.hpp:83-89 model, per launch
    # algorithmic bytes per matvec x matvecs timed, over the summed SBGEMV kernel time
    # (one launch per matvec on the device path; any column chunks sum to the same bytes)
    n_mv = 2 * args.steps
    t_gemv = (kms[1] + kms[2]) * 1e-3
    achieved = gemv_bytes * n_mv / t_gemv / 1e9 if t_gemv > 0 else None
    r2c_bytes = NM * NT * 8 + NM * nb * es  # F's big r2c: real in + TOSI spectrum out
    c2r_bytes = NM * nb * 16 + NM * NT * 8  # F*'s big c2r
    detail = {}
    for name, cls in (("sbgemv_n", 1), ("sbgemv_c", 2)):
        if kn[cls]:
            t = kms[cls] / args.steps * 1e-3
            detail[name] = {"ms_per_matvec": t * 1e3, "launches_per_matvec": kn[cls] / args.steps,
                            "gbs": gemv_bytes / t / 1e9, "frac": gemv_bytes / t / 1e9 / peak}
    if kn[0]:
        detail["r2c_all_ms_per_step"] = kms[0] / args.steps
    if kn[3]:
        detail["c2r_all_ms_per_step"] = kms[3] / args.steps
    detail["fft_big_phase_bytes"] = {"r2c_F": r2c_bytes, "c2r_Fstar": c2r_bytes}
    # FFT phase (all r2c + c2r launches of a step: F's big r2c and small c2r,
    # F*'s small r2c and big c2r) as HBM GB/s against the same peak
    small = ND * NT * 8 + ND * nb * es + ND * nb * 16 + ND * NT * 8
    if kn[0] and kn[3]:
        t_fft = (kms[0] + kms[3]) / args.steps * 1e-3
        fb = r2c_bytes + c2r_bytes + small
        detail["fft_phase"] = {"bytes_per_step": fb, "ms_per_step": t_fft * 1e3, "gbs": fb / t_fft / 1e9,
                               "frac": fb / t_fft / 1e9 / peak}
    share = (kms[1] + kms[2]) / ms if ms > 0 else None
    traffic = None
    nc = ncu_traffic()
    if nc and "sbgemv_dram_bytes_per_launch" in nc:
        traffic = nc["sbgemv_dram_bytes_per_launch"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic, "kernel": "sbgemv (N for F, C for F*)",
                "algorithmic_bytes_per_matvec": gemv_bytes, "peak_source": peak_src, "share_of_step": share,
                "detail": detail}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if cfg == "ddddd" else f"mixed:{cfg}", "data": "synthetic (reference uniform_fill, seeded)",
        "config": workload_config(world, cfg),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": ms_e2e / args.steps, "api": e2e_api},
        "e2e_blocking": {"value": 2 * args.steps * world / (ms_blk * 1e-3), "unit": UNIT,
                         "ms_per_step": ms_blk / args.steps,
                         "api": "fmv_matvec / fmv_matvec_partitioned (C ABI, blocking), pinned host buffers"},
        "gpu_launches": int(launches) * world,
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_block and cfg[2] in "ds":
        line["block"] = block_throughput(F, L, ctx, op, cfg, m_h, d_h, dev, stream)
    if rank == 0 and world == 1 and not args.no_dropin:
        line["e2e_dropin"] = dropin_e2e(cfg, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(col, m_h, d_h, cfg)
    return line


def dropin_e2e(cfg, args):
    """Second end-to-end figure: the reference's own C++ API (include/fftmv
    forward_matvec / adjoint_matvec with std::vector host vectors and
    PhaseTimings, build/fftmv_dropin_bench), host wall clock per step, in a
    separate process on the same GPU."""
    exe = os.path.join(HERE, "build", "fftmv_dropin_bench")
    if not os.path.exists(exe):
        return {"value": None, "unit": UNIT, "note": "build/fftmv_dropin_bench not built (make cli)"}
    try:
        r = subprocess.run([exe, str(NM), str(ND), str(NT), cfg, str(args.steps), str(max(3, args.warmup))],
                           capture_output=True, text=True, timeout=600)
        j = json.loads(r.stdout.strip().splitlines()[-1])
        return {"value": j["matvecs_per_s"], "unit": UNIT, "ms_per_step": j["ms_per_step"],
                "h2d_bytes_per_step": j["h2d_bytes_per_step"], "d2h_bytes_per_step": j["d2h_bytes_per_step"],
                "api": "C++ drop-in fftmv::forward_matvec / adjoint_matvec (reference signatures, pageable "
                       "std::vector I/O, PhaseTimings on), host wall clock"}
    except Exception as e:  # report, do not hide
        return {"value": None, "unit": UNIT, "note": f"dropin bench failed: {e}"}


def block_throughput(F, L, ctx, op, cfg, m_h, d_h, dev, stream, reps=5):
    """Extra (not the headline): the block (multi-RHS) matvec, SURVEY.md §8 f2 --
    K right-hand sides per call (8 for F, 4 for F*), the operator streamed once
    per call; device-resident I/O, per-RHS matvecs/s, CUDA events."""
    import torch

    from paper_2508_10202_b200 import _capi

    out = {}
    for kind, K, x_h, n_out in ((0, 8, m_h, ND * NT), (1, 4, d_h, NM * NT)):
        X = torch.from_numpy(np.tile(x_h, K)).to(dev)
        Y = torch.empty(K * n_out, dtype=torch.float64, device=dev)

        def call():
            _capi.check(L.fmv_matvec_block_async(ctx.handle, op.handle, kind, cfg.encode(), K,
                                                 ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Y.data_ptr())))
        for _ in range(2):
            call()
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            call()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out["F" if kind == 0 else "Fstar"] = {"rhs_per_call": K, "ms_per_call": ms, "matvecs_per_s": K / (ms * 1e-3)}
    out["note"] = "extra: block matvec (fmv_matvec_block), operator read once per call; not the headline value"
    return out


def cpu_baseline(col, m, d, cfg):
    try:
        R, op, t_setup = ref_setup(col)
        T = cpu_threads()
        t = R.throughput_mixed(op, cfg, m, d, T)
        lat_f = R.throughput(op, 0, cfg, m, 1, 1)
        return {"value": T / t, "unit": UNIT, "cores": T, "kind": "reference",
                "sample": (f"{T} threads concurrently, one matvec each (half F, half F*) on one shared C2 operator, "
                           f"reference headers compiled verbatim (oracle/_ref, FFTW API over MKL DFTI); "
                           f"1-thread F latency {lat_f:.2f}s; setup_operator {t_setup:.1f}s excluded")}
    except Exception as e:  # the reference .so is a checker; report why it is missing
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` without a launcher: re-exec as N ranks (one
    per GPU) under torch.distributed.run on 127.0.0.1, as the driver does."""
    import socket

    import torch

    n = torch.cuda.device_count()
    if n < args.gpus and os.environ.get("FMV_BENCH_SHARED_GPU") != "1":
        raise SystemExit(f"bench: --gpus {args.gpus} but only {n} visible GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # to stderr (NCCL_DEBUG_FILE): shows the communicator's nranks
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", default="ddddd")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-block", action="store_true", help="skip the block (multi-RHS) extra measurement")
    ap.add_argument("--no-dropin", action="store_true", help="skip the C++ drop-in e2e measurement")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5"],
                    help="c2: Nm=5000, Nd=100, Nt=1000 per GPU (default); c5: Nd=600 (48 GB fp64 operator per GPU)")
    args = ap.parse_args()
    global ND
    if args.workload == "c5":
        ND = 600
        args.no_cpu_baseline = True  # the reference needs ~70 GB host RAM and minutes of setup at C5
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        relaunch_under_torchrun(args)  # does not return
    # stdout carries exactly one JSON line: keep the real stdout for it and send
    # everything else written to fd 1 (NCCL's version banner, library prints)
    # to stderr
    json_out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    # test only (tests/test_gpu_multiproc.py): every rank on cuda:0, gloo for
    # the host-side collectives, the library's collectives through the NCCL
    # test transport (FMV_NCCL_LIB) -- checks the multi-rank flow of this
    # script on a one-GPU box; its timings mean nothing
    shared = os.environ.get("FMV_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else local_rank
    if "WORLD_SIZE" in os.environ and args.impl == "ours" and world != args.gpus and "--gpus" in " ".join(sys.argv):
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist

        if shared:
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            if torch.cuda.device_count() < world:
                raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} visible GPUs")
            if local_rank >= torch.cuda.device_count():
                raise SystemExit(f"bench: LOCAL_RANK {local_rank} has no GPU")
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.impl == "reference":
        line = run_reference_arm(args, rank, world)
    else:
        line = run_ours(args, rank, world, gpu)
    if rank == 0 and line is not None:
        print(json.dumps(line), file=json_out, flush=True)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
