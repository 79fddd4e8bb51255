"""B200-native FFTMatvec (sm_100a) -- drop-in for the reference FFTMatvec path.

See DESIGN.md. The compute lives in libfftmv_cuda.so (C ABI in
include/fftmv_cuda.h); this package is the host-side mirror of the reference
API (/root/reference/proj/include/fftmv): core types + pipeline (fftmv.py),
L1 kernels (kernels.py), the mixed-precision lab (preclab.py) and the 1 x p
partition (partition.py).
"""
from .fftmv import *  # noqa: F401,F403
from .fftmv import __all__ as _a1
from .kernels import *  # noqa: F401,F403
from .kernels import __all__ as _a2
from .preclab import *  # noqa: F401,F403
from .preclab import __all__ as _a3
from .partition import *  # noqa: F401,F403
from .partition import __all__ as _a4
from .vector_io import *  # noqa: F401,F403
from .vector_io import __all__ as _a5
from ._capi import FmvError, LIB_PATH, lib  # noqa: F401

__all__ = list(_a1) + list(_a2) + list(_a3) + list(_a4) + list(_a5) + ["lib", "LIB_PATH"]
