"""ctypes binding of libfftmv_cuda.so (include/fftmv_cuda.h).

The shared library is built in-tree by ``make lib`` (or ``__graft_entry__.build()``).
There is no fallback: if the library is missing or the device is not an
sm_100 part, every compute call raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_char_p, c_double, c_int, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# FMV_LIB_PATH: load an alternative build (A/B tuning runs); default is the in-tree library.
LIB_PATH = os.environ.get("FMV_LIB_PATH") or os.path.join(_HERE, "libfftmv_cuda.so")

FMV_OK, FMV_EINVAL, FMV_ECUDA, FMV_ENCCL, FMV_ENOMEM, FMV_EUNSUPPORTED = 0, 1, 2, 3, 4, 5
FORWARD, ADJOINT = 0, 1
GEMV_N, GEMV_T, GEMV_C = 0, 1, 2


class FmvError(RuntimeError):
    """Backend failure (std::runtime_error in the reference, fft.hpp:63)."""


class PhaseTimesC(ctypes.Structure):
    _fields_ = [("phase_s", c_double * 5), ("total_s", c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libfftmv_cuda.so once; raise loudly if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FmvError(f"{LIB_PATH} is not built; run `make lib` (or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "fmv_last_error": (c_char_p, []),
        "fmv_version": (c_char_p, []),
        "fmv_ctx_create": (c_int, [c_int, c_void_p, POINTER(c_void_p)]),
        "fmv_ctx_destroy": (c_int, [c_void_p]),
        "fmv_ctx_stream": (c_void_p, [c_void_p]),
        "fmv_ctx_launches": (c_uint64, [c_void_p]),
        "fmv_ctx_set_profiling": (c_int, [c_void_p, c_int]),
        "fmv_ctx_profile_read": (c_int, [c_void_p, POINTER(c_double), POINTER(c_uint64), c_int]),
        "fmv_synchronize": (c_int, [c_void_p]),
        "fmv_op_create": (c_int, [c_void_p, c_size_t, c_size_t, c_size_t, c_void_p, c_int, POINTER(c_void_p)]),
        "fmv_op_destroy": (c_int, [c_void_p]),
        "fmv_op_dims": (c_int, [c_void_p, POINTER(c_size_t), POINTER(c_size_t), POINTER(c_size_t)]),
        "fmv_op_materialize": (c_int, [c_void_p, c_void_p, c_char]),
        "fmv_op_has": (c_int, [c_void_p, c_char]),
        "fmv_op_download_bins": (c_int, [c_void_p, c_void_p, c_char, c_void_p]),
        "fmv_op_device_bytes": (c_size_t, [c_void_p]),
        "fmv_matvec": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p, c_int, POINTER(PhaseTimesC)]),
        "fmv_matvec_payload": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_char, c_void_p, c_void_p, c_int,
                                       POINTER(PhaseTimesC)]),
        "fmv_matvec_async": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p]),
        "fmv_matvec_host_async": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p]),
        "fmv_join": (c_int, [c_void_p]),
        "fmv_matvec_block": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_size_t, c_void_p, c_void_p, c_int]),
        "fmv_matvec_block_async": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_size_t, c_void_p, c_void_p]),
        "fmv_casts_performed": (c_uint64, []),
        "fmv_reset_cast_counter": (None, []),
        "fmv_sbgemv": (c_int, [c_void_p, c_int, c_char, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, c_void_p,
                               c_size_t, c_void_p, c_size_t, c_void_p, c_int, POINTER(c_int)]),
        "fmv_comm_unique_id": (c_int, [c_void_p]),
        "fmv_comm_init": (c_int, [c_void_p, c_int, c_int, c_void_p]),
        "fmv_comm_destroy": (c_int, [c_void_p]),
        "fmv_comm_size": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
        "fmv_matvec_partitioned": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p, c_int,
                                           POINTER(PhaseTimesC)]),
        "fmv_matvec_partitioned_async": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p]),
        "fmv_graph_create": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p, POINTER(c_void_p)]),
        "fmv_graph_launch": (c_int, [c_void_p]),
        "fmv_graph_destroy": (c_int, [c_void_p]),
        "fmv_comm_init_2d": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p]),
        "fmv_matvec_partitioned_2d": (c_int, [c_void_p, c_void_p, c_int, c_char_p, c_void_p, c_void_p, c_int]),
        "fmv_fft_r2c": (c_int, [c_void_p, c_size_t, c_size_t, c_char, c_void_p, c_void_p]),
        "fmv_fft_c2r": (c_int, [c_void_p, c_size_t, c_size_t, c_char, c_void_p, c_void_p]),
        "fmv_seed_stream": (c_uint64, [c_uint64, c_uint64]),
        "fmv_uniform_fill": (None, [c_size_t, c_uint64, c_double, c_double, c_void_p]),
        "fmv_non_representable_fill": (c_int, [c_size_t, c_uint64, c_void_p]),
        "fmv_relative_error": (c_int, [c_size_t, c_void_p, c_void_p, POINTER(c_double)]),
        "fmv_host_copy": (c_int, [c_void_p, c_void_p, c_size_t]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    return [
        "fmv_last_error", "fmv_version", "fmv_ctx_create", "fmv_ctx_destroy", "fmv_ctx_stream", "fmv_ctx_launches",
        "fmv_ctx_set_profiling", "fmv_ctx_profile_read", "fmv_synchronize", "fmv_op_create", "fmv_op_destroy",
        "fmv_op_dims", "fmv_op_materialize", "fmv_op_has", "fmv_op_download_bins", "fmv_op_device_bytes",
        "fmv_matvec", "fmv_matvec_async", "fmv_casts_performed", "fmv_reset_cast_counter", "fmv_sbgemv",
        "fmv_comm_unique_id", "fmv_comm_init", "fmv_comm_destroy", "fmv_matvec_partitioned", "fmv_seed_stream",
        "fmv_uniform_fill", "fmv_non_representable_fill", "fmv_relative_error", "fmv_fft_r2c", "fmv_fft_c2r",
        "fmv_matvec_block", "fmv_matvec_block_async", "fmv_comm_init_2d", "fmv_matvec_partitioned_2d",
        "fmv_graph_create", "fmv_graph_launch", "fmv_graph_destroy", "fmv_matvec_payload", "fmv_comm_size",
        "fmv_matvec_partitioned_async", "fmv_host_copy", "fmv_matvec_host_async", "fmv_join",
    ]


def check(rc: int) -> None:
    """Map C ABI return codes to the reference's exception types."""
    if rc == FMV_OK:
        return
    msg = lib().fmv_last_error().decode(errors="replace")
    if rc == FMV_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    raise FmvError(f"[code {rc}] {msg}")
