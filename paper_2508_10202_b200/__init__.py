"""B200-native FFTMatvec (sm_100a) -- drop-in for the reference FFTMatvec path.

See DESIGN.md. The compute lives in libfftmv_cuda.so (C ABI in
include/fftmv_cuda.h); this package is the host-side mirror of the reference
API (/root/reference/proj/include/fftmv).
"""
from .fftmv import *  # noqa: F401,F403
from .fftmv import __all__ as _fftmv_all
from ._capi import FmvError, LIB_PATH, lib  # noqa: F401

__all__ = list(_fftmv_all) + ["lib", "LIB_PATH"]
