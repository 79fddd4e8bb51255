"""Mixed-precision experiment engine on B200 (sweep.hpp:1-233): the 32-config
sweep, error metric, Pareto front, optimal-config choice and CSV/JSON reports.

The selection logic is the reference's verbatim in behaviour; what changes is
the clock: rows are timed with CUDA events around device-resident matvecs
(``timing="device"``, default) or wall-clock around the blocking host-I/O call
(``timing="host"``, the reference's convention, sweep.hpp:84-92).
"""
from __future__ import annotations

import ctypes
import json
import math
import time
from dataclasses import dataclass, field
from typing import Callable, Iterable, List, Optional, Sequence

import numpy as np

from ._capi import check, lib
from .fftmv import (MatvecKind, PrecisionConfig, ProblemDims, SpectralOperator, enumerate_configs,
                    materialize_single, parse_precision_config, relative_error, run_pipeline)

__all__ = ["ConfigResult", "sweep_configs", "sweep_operator", "dominates", "pareto_front", "optimal_config",
           "SweepReport", "make_report", "kind_name", "sweep_csv_header", "to_csv", "to_json", "parse_sweep_csv"]


@dataclass
class ConfigResult:
    """sweep.hpp:62-68."""

    config: PrecisionConfig
    mean_s: float = 0.0
    min_s: float = 0.0
    max_s: float = 0.0
    rel_error: float = 0.0


def sweep_configs(run_cfg: Callable, repetitions: int, warmup: int,
                  configs: Optional[Sequence[PrecisionConfig]] = None,
                  timer: Optional[Callable] = None) -> List[ConfigResult]:
    """sweep.hpp:74-104. ``run_cfg(cfg) -> np.ndarray``; the first config must
    be "ddddd" (baseline). ``timer(cfg) -> (output, seconds)`` optionally
    replaces the wall clock (device timing)."""
    if repetitions < 1:
        raise ValueError("sweep_configs: repetitions must be >= 1")
    if warmup < 0:
        raise ValueError("sweep_configs: warmup must be >= 0")
    configs = list(configs) if configs is not None else enumerate_configs()
    rows: List[ConfigResult] = []
    baseline = None
    for cfg in configs:
        for _ in range(warmup):
            run_cfg(cfg)
        row = ConfigResult(cfg, min_s=math.inf)
        total = 0.0
        out = None
        for _ in range(repetitions):
            if timer is None:
                t0 = time.perf_counter()
                out = run_cfg(cfg)
                dt = time.perf_counter() - t0
            else:
                out, dt = timer(cfg)
            total += dt
            row.min_s = min(row.min_s, dt)
            row.max_s = max(row.max_s, dt)
        row.mean_s = total / repetitions
        if baseline is None:
            baseline = np.array(out, copy=True)
        row.rel_error = 0.0 if cfg == PrecisionConfig.all_double() else relative_error(out, baseline)
        rows.append(row)
    return rows


def sweep_operator(op: SpectralOperator, inp, kind: MatvecKind, repetitions: int, warmup: int,
                   configs: Optional[Sequence[PrecisionConfig]] = None, timing: str = "device") -> List[ConfigResult]:
    """sweep.hpp:108-119 on the GPU. Single (and, if swept, half) bins are
    materialized up front so no setup cost leaks into the timed region."""
    import torch

    materialize_single(op)
    configs = list(configs) if configs is not None else enumerate_configs()
    if any(c.render()[2] == "h" for c in configs):
        op.ensure_half()
    n_in = (op.dims.n_m if kind == MatvecKind.Forward else op.dims.n_d) * op.dims.n_t
    n_out = (op.dims.n_d if kind == MatvecKind.Forward else op.dims.n_m) * op.dims.n_t
    x = np.ascontiguousarray(inp, dtype=np.float64).reshape(-1)
    if x.size != n_in:
        raise ValueError("sweep_configs: bad input length")
    if timing == "host":
        return sweep_configs(lambda c: run_pipeline(op, kind, x, c)[0], repetitions, warmup, configs)
    ctx = op.ctx
    dev = torch.device("cuda", ctx.device)
    xd = torch.from_numpy(x).to(dev)
    yd = torch.empty(n_out, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=dev)
    L = lib()

    def launch(cfg):
        check(L.fmv_matvec_async(ctx.handle, op.handle, int(kind), cfg.render().encode(),
                                 ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr())))

    def run(cfg):
        launch(cfg)
        ctx.synchronize()
        return yd.cpu().numpy()

    def timer(cfg):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch(cfg)
        e1.record(stream)
        e1.synchronize()
        return yd.cpu().numpy(), e0.elapsed_time(e1) * 1e-3

    return sweep_configs(run, repetitions, warmup, configs, timer=timer)


def dominates(r: ConfigResult, q: ConfigResult) -> bool:
    """sweep.hpp:121-125."""
    return (r.mean_s <= q.mean_s and r.rel_error <= q.rel_error and
            (r.mean_s < q.mean_s or r.rel_error < q.rel_error))


def pareto_front(results: Sequence[ConfigResult]) -> List[ConfigResult]:
    """sweep.hpp:127-139: non-dominated rows, input order preserved."""
    return [r for r in results if not any(dominates(q, r) for q in results)]


def optimal_config(results: Sequence[ConfigResult], tol: float) -> PrecisionConfig:
    """sweep.hpp:143-156: fastest with error <= tol; ties -> lower error -> smaller string."""
    if not tol > 0.0:
        raise ValueError("optimal_config: tolerance must be > 0")
    best = None
    for r in results:
        if r.rel_error > tol:
            continue
        if (best is None or r.mean_s < best.mean_s or
                (r.mean_s == best.mean_s and (r.rel_error < best.rel_error or
                                              (r.rel_error == best.rel_error and
                                               r.config.render() < best.config.render())))):
            best = r
    if best is None:
        raise ValueError("optimal_config: no result within tolerance")
    return best.config


@dataclass
class SweepReport:
    """sweep.hpp:158-166."""

    dims: ProblemDims
    kind: MatvecKind = MatvecKind.Forward
    repetitions: int = 0
    tolerance: float = 0.0
    rows: List[ConfigResult] = field(default_factory=list)
    chosen: Optional[PrecisionConfig] = None


def kind_name(k: MatvecKind) -> str:
    return "forward" if k == MatvecKind.Forward else "adjoint"


def make_report(dims: ProblemDims, kind: MatvecKind, repetitions: int, tol: float,
                rows: List[ConfigResult]) -> SweepReport:
    """sweep.hpp:169-179."""
    return SweepReport(dims, kind, repetitions, tol, list(rows), optimal_config(rows, tol))


def sweep_csv_header() -> str:
    return "config,mean_s,min_s,max_s,rel_error"


def to_csv(rep: SweepReport) -> str:
    """sweep.hpp:183-191 (17 significant digits)."""
    lines = [sweep_csv_header()]
    for r in rep.rows:
        lines.append(f"{r.config.render()},{r.mean_s:.17g},{r.min_s:.17g},{r.max_s:.17g},{r.rel_error:.17g}")
    return "\n".join(lines) + "\n"


def to_json(rep: SweepReport) -> dict:
    """sweep.hpp:193-208."""
    return {
        "dims": {"n_m": rep.dims.n_m, "n_d": rep.dims.n_d, "n_t": rep.dims.n_t},
        "kind": kind_name(rep.kind),
        "repetitions": rep.repetitions,
        "tolerance": rep.tolerance,
        "chosen": rep.chosen.render() if rep.chosen else None,
        "rows": [{"config": r.config.render(), "mean_s": r.mean_s, "min_s": r.min_s, "max_s": r.max_s,
                  "rel_error": r.rel_error} for r in rep.rows],
    }


def parse_sweep_csv(text: str) -> List[ConfigResult]:
    """sweep.hpp:211-233 (header optional, '#' lines skipped)."""
    rows = []
    for line in text.splitlines():
        if not line or line.startswith("#") or line == sweep_csv_header():
            continue
        parts = line.split(",")
        cfg = parse_precision_config(parts[0])
        names = ["mean_s", "min_s", "max_s", "rel_error"]
        vals = []
        for i, nm in enumerate(names):
            if len(parts) <= i + 1 or parts[i + 1] == "":
                raise ValueError(f"sweep csv: missing {nm}")
            vals.append(float(parts[i + 1]))
        rows.append(ConfigResult(cfg, *vals))
    return rows
