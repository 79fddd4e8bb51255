"""Front-ends of the L1 numerical kernels: batched real FFTs (fft.hpp:32-164)
and strided-batched GEMV (gemv.hpp:33-240), running the sm_100a kernels.

Inputs may be numpy arrays (copied to the device and back) or CUDA torch
tensors (used in place). Shapes/strides follow the reference exactly.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from ._capi import check, lib
from .fftmv import Precision, _is_cuda_tensor, default_context

__all__ = ["FftDirection", "FftPlan", "forward_real_batched", "inverse_real_batched", "GemvMode", "TilingParams",
           "KernelChoice", "select_kernel", "effective_bandwidth", "gemv_batched"]


class FftDirection(enum.IntEnum):
    Forward = 0
    Inverse = 1


@dataclass(frozen=True)
class FftPlan:
    """fft.hpp:32-95 (geometry only: the B200 kernels need no planner state
    beyond the cached twiddle tables inside the library)."""

    length: int
    batch: int
    precision: Precision
    direction: FftDirection

    def __post_init__(self):
        if self.length < 2 or self.length % 2:
            raise ValueError("FftPlan: length must be even and >= 2")
        if self.batch < 1:
            raise ValueError("FftPlan: batch must be >= 1")

    def n_bins(self) -> int:
        return self.length // 2 + 1


def _run_fft(fn, plan: FftPlan, x, n_in, in_dt, n_out, out_dt):
    import torch

    ctx = default_context()
    prec = b"d" if plan.precision == Precision.Double else b"s"
    if _is_cuda_tensor(x):
        xin = x.contiguous()
        if xin.numel() != n_in:
            raise ValueError(f"FFT: length mismatch, got {xin.numel()} scalars, expected {n_in}")
        out = torch.empty(n_out, dtype=out_dt, device=xin.device)
        torch.cuda.current_stream(xin.device).synchronize()
        check(fn(ctx.handle, plan.length, plan.batch, prec, ctypes.c_void_p(xin.data_ptr()),
                 ctypes.c_void_p(out.data_ptr())))
        ctx.synchronize()
        return out
    a = np.ascontiguousarray(x, dtype=in_dt).reshape(-1)
    if a.size != n_in:
        raise ValueError(f"FFT: length mismatch, got {a.size} scalars, expected {n_in}")
    dev = torch.from_numpy(a.view(np.float64) if a.dtype == np.complex128 else
                           a.view(np.float32) if a.dtype == np.complex64 else a).cuda()
    out = torch.empty(n_out, dtype=out_dt, device=dev.device)
    torch.cuda.current_stream(dev.device).synchronize()
    check(fn(ctx.handle, plan.length, plan.batch, prec, ctypes.c_void_p(dev.data_ptr()),
             ctypes.c_void_p(out.data_ptr())))
    ctx.synchronize()
    return out.cpu().numpy()


def forward_real_batched(plan: FftPlan, series):
    """fft.hpp:110-125: batch x length reals -> batch x n_bins complex (unnormalized)."""
    import torch

    if plan.direction != FftDirection.Forward:
        raise ValueError("FFT: plan direction mismatch")
    dbl = plan.precision == Precision.Double
    rdt = np.float64 if dbl else np.float32
    n_out = 2 * plan.n_bins() * plan.batch
    out = _run_fft(lib().fmv_fft_r2c, plan, series, plan.length * plan.batch, rdt, n_out,
                   torch.float64 if dbl else torch.float32)
    if isinstance(out, np.ndarray):
        return out.view(np.complex128 if dbl else np.complex64)
    return out


def inverse_real_batched(plan: FftPlan, bins):
    """fft.hpp:130-148: the true inverse (1/length included)."""
    import torch

    if plan.direction != FftDirection.Inverse:
        raise ValueError("FFT: plan direction mismatch")
    dbl = plan.precision == Precision.Double
    cdt = np.complex128 if dbl else np.complex64
    if _is_cuda_tensor(bins):
        n_in = 2 * plan.n_bins() * plan.batch
    else:
        bins = np.ascontiguousarray(bins, dtype=cdt).reshape(-1)
        if bins.size != plan.n_bins() * plan.batch:
            raise ValueError(f"FFT: length mismatch, got {bins.size} scalars, expected {plan.n_bins() * plan.batch}")
        bins = bins.view(np.float64 if dbl else np.float32)
        n_in = bins.size
    return _run_fft(lib().fmv_fft_c2r, plan, bins, n_in, np.float64 if dbl else np.float32,
                    plan.length * plan.batch, torch.float64 if dbl else torch.float32)


# ------------------------------------------------------------------ GEMV ---
class GemvMode(enum.IntEnum):
    NoTrans = 0
    Trans = 1
    ConjTrans = 2


class KernelChoice(enum.IntEnum):
    Naive = 0
    Tiled = 1


@dataclass(frozen=True)
class TilingParams:
    """gemv.hpp:63-68. Kept for signature parity; the B200 SBGEMV sizes its
    own shared-memory stages."""

    col_tile: int = 256
    row_chunk: int = 64
    dispatch_ratio: float = 1.0
    row_cutoff: int = 1024


def select_kernel(m: int, n: int, mode: GemvMode, p: TilingParams = TilingParams()) -> KernelChoice:
    """gemv.hpp:74-79 (the reference's CPU dispatch rule, reported for parity)."""
    if mode == GemvMode.NoTrans:
        return KernelChoice.Naive
    if float(m) < p.dispatch_ratio * float(n) and m <= p.row_cutoff:
        return KernelChoice.Tiled
    return KernelChoice.Naive


def effective_bandwidth(m: int, n: int, batch: int, elem_bytes: int, seconds: float) -> float:
    """gemv.hpp:83-89: batch*(m*n+m+n)*elem_bytes/seconds/1e9 GB/s."""
    if not seconds > 0.0:
        raise ValueError("effective_bandwidth: seconds must be > 0")
    elems = float(m) * float(n) + float(m) + float(n)
    return float(batch) * elems * float(elem_bytes) / seconds / 1e9


_DT = {"s": (np.float32, 4), "d": (np.float64, 8), "c": (np.complex64, 8), "z": (np.complex128, 16)}


def gemv_batched(mode: GemvMode, dtype: str, m: int, n: int, batch: int, lda: int, stride_a: int, A, stride_x: int,
                 x, stride_y: int, y=None, force_simple: bool = False, ctx=None):
    """y_b = op(A_b) x_b on the GPU (gemv.hpp:206-240 semantics). A, x, y are
    CUDA torch tensors (any dtype viewable as the element type) or numpy
    arrays. Returns (y, kernel_used) with kernel_used 0 = staged TMA kernel,
    1 = simple kernel."""
    import torch

    ctx = ctx or default_context()
    if m == 0 or n == 0 or batch == 0:
        raise ValueError("gemv: empty matrix batch")
    ylen = n if mode != GemvMode.NoTrans else m
    host = not _is_cuda_tensor(A)
    if host:
        npdt, es = _DT[dtype]
        a_np = np.ascontiguousarray(A, dtype=npdt).reshape(-1)
        x_np = np.ascontiguousarray(x, dtype=npdt).reshape(-1)
        y_np = np.zeros((batch - 1) * stride_y + ylen, dtype=npdt) if y is None else np.array(y, dtype=npdt)

        def dev(arr):
            buf = torch.zeros(arr.nbytes + 64, dtype=torch.uint8, device="cuda")
            buf[: arr.nbytes].copy_(torch.from_numpy(arr.view(np.uint8)))
            return buf

        A_d, x_d, y_d = dev(a_np), dev(x_np), dev(y_np)
    else:
        A_d, x_d, y_d = A, x, y
    used = ctypes.c_int(-1)
    torch.cuda.synchronize()
    check(lib().fmv_sbgemv(ctx.handle, int(mode), dtype.encode(), m, n, batch, lda, stride_a,
                           ctypes.c_void_p(A_d.data_ptr()), stride_x, ctypes.c_void_p(x_d.data_ptr()), stride_y,
                           ctypes.c_void_p(y_d.data_ptr()), 1 if force_simple else 0, ctypes.byref(used)))
    ctx.synchronize()
    if host:
        out = y_d[: y_np.nbytes].cpu().numpy().view(y_np.dtype).copy()
        return out, used.value
    return y_d, used.value
