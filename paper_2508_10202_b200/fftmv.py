"""Host-side mirror of the reference FFTMatvec API (namespace ``fftmv``,
/root/reference/proj/include/fftmv/*.hpp), backed by libfftmv_cuda.so.

Names, argument meaning and error behaviour follow the reference so that the
parity tests read like the reference's own: ``ProblemDims`` (dims.hpp:10-26),
``PrecisionConfig`` / ``parse_precision_config`` / ``enumerate_configs``
(config.hpp:14-65), ``BlockColumn`` / ``SpectralOperator`` / ``setup_operator``
/ ``materialize_single`` (operator.hpp:30-125), ``forward_matvec`` /
``adjoint_matvec`` / ``PhaseTimings`` / ``MatvecResult`` (matvec.hpp:42-318),
``BlockVector`` / ``reorder`` (block_vector.hpp:14-93), fills
(random_fill.hpp:17-32, sweep.hpp:32-46). ``std::invalid_argument`` maps to
``ValueError``; backend failures raise ``FmvError``.

All compute runs in sm_100a kernels through the C ABI. Host vectors are
numpy float64 arrays; CUDA torch tensors are accepted for device-resident I/O.
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import FmvError, check, lib

__all__ = [
    "ProblemDims", "Precision", "PrecisionConfig", "parse_precision_config", "enumerate_configs",
    "precision_char", "Layout", "Domain", "BlockVector", "reorder", "BlockColumn", "SpectralOperator",
    "setup_operator", "materialize_single", "MatvecKind", "PhaseTimings", "MatvecResult", "phase_name",
    "forward_matvec", "adjoint_matvec", "run_pipeline", "Context", "default_context", "casts_performed",
    "reset_cast_counter", "uniform_fill", "seed_stream", "non_representable_fill", "relative_error", "FmvError",
    "matvec_block", "forward_matvec_block", "adjoint_matvec_block", "MatvecGraph", "matvec_host_async",
]


# ------------------------------------------------------------------ dims ---
@dataclass(frozen=True)
class ProblemDims:
    """dims.hpp:10-26."""

    n_m: int
    n_d: int
    n_t: int

    def __post_init__(self):
        if self.n_m < 1 or self.n_d < 1 or self.n_t < 1:
            raise ValueError("ProblemDims: all extents must be >= 1")

    def fft_len(self) -> int:
        return 2 * self.n_t

    def n_bins(self) -> int:
        return self.n_t + 1


# ------------------------------------------------------------- precision ---
class Precision(enum.IntEnum):
    """precision.hpp:15; Half is this project's fp16 extension and
    SingleAccDouble ('m', SBGEMV slot only) its fp32-storage / fp64-accumulate
    SBGEMV variant, appended so Single=0 / Double=1 keep
    their values."""

    Single = 0
    Double = 1
    Half = 2
    SingleAccDouble = 3


_P2C = {Precision.Double: "d", Precision.Single: "s", Precision.Half: "h", Precision.SingleAccDouble: "m"}
_C2P = {v: k for k, v in _P2C.items()}


def precision_char(p: Precision) -> str:
    return _P2C[Precision(p)]


@dataclass(frozen=True)
class PrecisionConfig:
    """config.hpp:14-33: [0] pad/broadcast, [1] FFT, [2] SBGEMV, [3] IFFT, [4] unpad/reduce."""

    phase: tuple = (Precision.Double,) * 5

    def __getitem__(self, i: int) -> Precision:
        return self.phase[i]

    def render(self) -> str:
        return "".join(_P2C[p] for p in self.phase)

    @staticmethod
    def all_double() -> "PrecisionConfig":
        return PrecisionConfig()

    def __str__(self) -> str:
        return self.render()


def parse_precision_config(s: str, allow_half: bool = True) -> PrecisionConfig:
    """config.hpp:36-51 (errors name the 1-based position); the extensions
    (allow_half): 'h' (fp16) at positions 1, 3, 5 and 'm' (fp32 storage, fp64
    accumulation) at position 3."""
    if len(s) != 5:
        raise ValueError(f"precision config must be exactly 5 characters, got {len(s)}")
    out = []
    for i, ch in enumerate(s):
        ok = ch in ("d", "s") or (allow_half and ((ch == "h" and i in (0, 2, 4)) or (ch == "m" and i == 2)))
        if not ok:
            exp = "'d' or 's'" + (" (or 'h' at positions 1, 3, 5, 'm' at position 3)" if allow_half else "")
            raise ValueError(f"precision config: invalid character '{ch}' at position {i + 1} (expected {exp})")
        out.append(_C2P[ch])
    return PrecisionConfig(tuple(out))


def enumerate_configs(include_half: bool = False) -> list:
    """config.hpp:55-65: the 32 {d,s} configs in lexicographic order ('d' < 's').
    include_half=True appends the extension variants ('h' at phases 1/3/5,
    'm' at phase 3), ordered the same way, after the 32 reference configs."""
    allc = []
    for bits in range(32):
        allc.append(PrecisionConfig(tuple(Precision.Single if (bits >> (4 - i)) & 1 else Precision.Double
                                          for i in range(5))))
    if include_half:
        seen = {c.render() for c in allc}
        import itertools

        for combo in itertools.product("dsh", "ds", "dshm", "ds", "dsh"):
            s = "".join(combo)
            if s not in seen:
                allc.append(parse_precision_config(s))
    return allc


def _cfg_str(cfg) -> str:
    if isinstance(cfg, PrecisionConfig):
        return cfg.render()
    if isinstance(cfg, str):
        return parse_precision_config(cfg).render()
    raise TypeError("cfg must be a PrecisionConfig or a 5-char string")


# --------------------------------------------------------- block vectors ---
class Layout(enum.IntEnum):
    SOTI = 0
    TOSI = 1


class Domain(enum.IntEnum):
    Time = 0
    Frequency = 1


@dataclass
class BlockVector:
    """block_vector.hpp:26-63 (one buffer: ``data`` is float64 or float32)."""

    space_extent: int
    time_extent: int
    layout: Layout = Layout.SOTI
    precision: Precision = Precision.Double
    domain: Domain = Domain.Time
    data: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def elements(self) -> int:
        return self.space_extent * self.time_extent

    def scalars_per_element(self) -> int:
        return 2 if self.domain == Domain.Frequency else 1

    def scalar_count(self) -> int:
        return self.elements() * self.scalars_per_element()

    @property
    def f64(self) -> np.ndarray:
        return self.data

    def validate(self) -> None:
        if self.space_extent == 0 or self.time_extent == 0:
            raise ValueError("BlockVector: zero extent")
        n = self.scalar_count()
        if self.data.size != n:
            raise ValueError(f"BlockVector: buffer length {self.data.size} does not match extents ({n} scalars)")

    @staticmethod
    def time_double(space: int, time: int, data, layout: Layout = Layout.SOTI) -> "BlockVector":
        arr = data if _is_cuda_tensor(data) else np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        v = BlockVector(space, time, layout, Precision.Double, Domain.Time, arr)
        if not _is_cuda_tensor(arr):
            v.validate()
        return v


def reorder(v: BlockVector, target: Layout) -> BlockVector:
    """block_vector.hpp:79-93: bitwise relayout SOTI <-> TOSI."""
    v.validate()
    if v.layout == target:
        return BlockVector(v.space_extent, v.time_extent, v.layout, v.precision, v.domain, v.data.copy())
    outer = v.space_extent if v.layout == Layout.SOTI else v.time_extent
    inner = v.time_extent if v.layout == Layout.SOTI else v.space_extent
    c = v.scalars_per_element()
    out = v.data.reshape(outer, inner, c).transpose(1, 0, 2).copy().reshape(-1)
    return BlockVector(v.space_extent, v.time_extent, target, v.precision, v.domain, out)


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and hasattr(x, "data_ptr") and bool(x.is_cuda)


# ------------------------------------------------------------------ ctx ----
class Context:
    """One device, one CUDA stream, a grow-only workspace (fmv_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = ctypes.c_void_p()
        check(lib().fmv_ctx_create(device, ctypes.c_void_p(stream) if stream else None, ctypes.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream_ptr(self) -> int:
        return lib().fmv_ctx_stream(self.handle) or 0

    def launches(self) -> int:
        return int(lib().fmv_ctx_launches(self.handle))

    def set_profiling(self, on: bool) -> None:
        check(lib().fmv_ctx_set_profiling(self.handle, 1 if on else 0))

    def profile_read(self, reset: bool = True):
        ms = (ctypes.c_double * 5)()
        n = (ctypes.c_uint64 * 5)()
        check(lib().fmv_ctx_profile_read(self.handle, ms, n, 1 if reset else 0))
        return list(ms), list(n)

    def synchronize(self) -> None:
        check(lib().fmv_synchronize(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().fmv_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


_ctx_lock = threading.Lock()
_ctx_by_thread: dict = {}


def default_context(device: int = 0) -> Context:
    """Per-(thread, device) context: contexts are single-threaded, operators shared."""
    key = (threading.get_ident(), device)
    with _ctx_lock:
        c = _ctx_by_thread.get(key)
        if c is None:
            c = Context(device)
            _ctx_by_thread[key] = c
        return c


# ------------------------------------------------------------- operator ----
@dataclass
class BlockColumn:
    """operator.hpp:30-54: Nt blocks of Nd x Nm, column-major within a block."""

    dims: ProblemDims
    data: np.ndarray

    def __post_init__(self):
        if not _is_cuda_tensor(self.data):
            self.data = np.ascontiguousarray(self.data, dtype=np.float64).reshape(-1)
        n = self.dims.n_t * self.dims.n_d * self.dims.n_m
        size = self.data.numel() if _is_cuda_tensor(self.data) else self.data.size
        if size != n:
            raise ValueError("BlockColumn: buffer length does not match dims")

    def block_elems(self) -> int:
        return self.dims.n_d * self.dims.n_m

    def at(self, t: int, i: int, j: int) -> float:
        return float(self.data[t * self.block_elems() + i + j * self.dims.n_d])

    @staticmethod
    def zeros(d: ProblemDims) -> "BlockColumn":
        return BlockColumn(d, np.zeros(d.n_t * d.n_d * d.n_m))


class SpectralOperator:
    """operator.hpp:56-87: the nb = Nt+1 frequency-bin matrices, device-resident.

    ``bins_double`` is downloaded on demand (the reference keeps it on host,
    operator.hpp:59); ``ensure_single`` materializes the fp32 copy on device.
    """

    def __init__(self, handle: ctypes.c_void_p, dims: ProblemDims, ctx: Context):
        self._h = handle
        self.dims = dims
        self.ctx = ctx

    @property
    def handle(self):
        return self._h

    def bin_elems(self) -> int:
        return self.dims.n_d * self.dims.n_m

    @property
    def bins_double(self) -> np.ndarray:
        nb = self.dims.n_bins()
        out = np.empty(nb * self.bin_elems(), dtype=np.complex128)
        check(lib().fmv_op_download_bins(self.ctx.handle, self._h, b"d", out.ctypes.data))
        return out

    def bins_single(self) -> np.ndarray:
        nb = self.dims.n_bins()
        out = np.empty(nb * self.bin_elems(), dtype=np.complex64)
        check(lib().fmv_op_download_bins(self.ctx.handle, self._h, b"s", out.ctypes.data))
        return out

    def has_single(self) -> bool:
        return bool(lib().fmv_op_has(self._h, b"s"))

    def ensure_single(self) -> "SpectralOperator":
        check(lib().fmv_op_materialize(self.ctx.handle, self._h, b"s"))
        return self

    def ensure_half(self) -> "SpectralOperator":
        check(lib().fmv_op_materialize(self.ctx.handle, self._h, b"h"))
        return self

    def device_bytes(self) -> int:
        return int(lib().fmv_op_device_bytes(self._h))

    def close(self) -> None:
        if self._h:
            lib().fmv_op_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def setup_operator(col: BlockColumn, ctx: Optional[Context] = None) -> SpectralOperator:
    """operator.hpp:99-125 on the GPU (fp64 r2c of every padded series)."""
    ctx = ctx or default_context()
    d = col.dims
    h = ctypes.c_void_p()
    if _is_cuda_tensor(col.data):
        check(lib().fmv_op_create(ctx.handle, d.n_m, d.n_d, d.n_t, ctypes.c_void_p(col.data.data_ptr()), 1,
                                  ctypes.byref(h)))
    else:
        check(lib().fmv_op_create(ctx.handle, d.n_m, d.n_d, d.n_t, col.data.ctypes.data, 0, ctypes.byref(h)))
    return SpectralOperator(h, d, ctx)


def materialize_single(op: SpectralOperator) -> SpectralOperator:
    """operator.hpp:90-93."""
    return op.ensure_single()


# ------------------------------------------------------------- pipeline ----
class MatvecKind(enum.IntEnum):
    Forward = 0
    Adjoint = 1


_PHASES = ("pad", "fft", "sbgemv", "ifft", "unpad")


def phase_name(i: int) -> str:
    """matvec.hpp:53-56."""
    return _PHASES[i]


@dataclass
class PhaseTimings:
    """matvec.hpp:42-51 (seconds; see fftmv_cuda.h for the fused attribution)."""

    phase_s: list = field(default_factory=lambda: [0.0] * 5)
    total_s: float = 0.0

    def __iadd__(self, o: "PhaseTimings") -> "PhaseTimings":
        self.phase_s = [a + b for a, b in zip(self.phase_s, o.phase_s)]
        self.total_s += o.total_s
        return self


@dataclass
class MatvecResult:
    output: BlockVector
    timings: PhaseTimings


def _check_input(op: SpectralOperator, v: BlockVector, forward: bool) -> None:
    """matvec.hpp:291-299."""
    n_in = op.dims.n_m if forward else op.dims.n_d
    if v.precision != Precision.Double:
        raise ValueError("matvec: input must be double precision")
    if v.domain != Domain.Time or v.layout != Layout.SOTI:
        raise ValueError("matvec: input must be a time-domain SOTI vector")
    if v.space_extent != n_in or v.time_extent != op.dims.n_t:
        raise ValueError("matvec: input extents do not match operator dims")
    if not _is_cuda_tensor(v.data):
        v.validate()


_PAYLOAD_DTYPES = {"d": np.float64, "s": np.float32, "h": np.float16}


def run_pipeline(op: SpectralOperator, kind: MatvecKind, inp, cfg="ddddd", ctx: Optional[Context] = None,
                 timings: bool = True, payload: Optional[str] = None):
    """matvec.hpp:233-289: returns (output, PhaseTimings). ``inp`` is a float64
    numpy array (host I/O) or a CUDA float64 torch tensor (device I/O).

    Host I/O always runs the overlapped schedule (input / output copies in
    column chunks beside the SBGEMV); ``timings=False`` skips the CUDA-event
    bookkeeping (``times = NULL`` at the C ABI) and returns zero timings.
    ``payload`` = 'd' / 's' / 'h': ``inp`` is a broadcast payload already
    rounded to cfg[0] and stored in that precision (float64 / float32 /
    float16 numpy array, matvec.hpp:240 ``payload``; partition.hpp:198-212)."""
    ctx = ctx or op.ctx
    fwd = kind == MatvecKind.Forward
    n_in = (op.dims.n_m if fwd else op.dims.n_d) * op.dims.n_t
    n_out = (op.dims.n_d if fwd else op.dims.n_m) * op.dims.n_t
    cs = _cfg_str(cfg).encode()
    t = _capi.PhaseTimesC()
    tp = ctypes.byref(t) if timings else None
    if payload is not None:
        if payload not in _PAYLOAD_DTYPES:
            raise ValueError("run_pipeline: payload precision must be 'd', 's' or 'h'")
        x = np.ascontiguousarray(inp, dtype=_PAYLOAD_DTYPES[payload]).reshape(-1)
        if x.size != n_in:
            raise ValueError("matvec: input length does not match operator dims")
        out = np.empty(n_out, dtype=np.float64)
        check(lib().fmv_matvec_payload(ctx.handle, op.handle, int(kind), cs, payload.encode(), x.ctypes.data,
                                       out.ctypes.data, 0, tp))
    elif _is_cuda_tensor(inp):
        import torch

        if inp.dtype != torch.float64 or inp.numel() != n_in:
            raise ValueError("matvec: input length does not match operator dims")
        x = inp.contiguous()
        out = torch.empty(n_out, dtype=torch.float64, device=x.device)
        torch.cuda.current_stream(x.device).synchronize()
        check(lib().fmv_matvec(ctx.handle, op.handle, int(kind), cs, ctypes.c_void_p(x.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()), 1, tp))
    else:
        x = np.ascontiguousarray(inp, dtype=np.float64).reshape(-1)
        if x.size != n_in:
            raise ValueError("matvec: input length does not match operator dims")
        out = np.empty(n_out, dtype=np.float64)
        check(lib().fmv_matvec(ctx.handle, op.handle, int(kind), cs, x.ctypes.data, out.ctypes.data, 0, tp))
    return out, PhaseTimings(list(t.phase_s), t.total_s)


def forward_matvec(op: SpectralOperator, m: BlockVector, cfg="ddddd", tiling=None,
                   timings: bool = True) -> MatvecResult:
    """matvec.hpp:305-310: d = F m. ``tiling`` (TilingParams) is accepted for
    signature parity and ignored: the B200 kernels pick their own tiles.
    ``timings=False``: no PhaseTimings bookkeeping (zeros returned)."""
    if not isinstance(m, BlockVector):
        m = BlockVector.time_double(op.dims.n_m, op.dims.n_t, m)
    _check_input(op, m, True)
    out, t = run_pipeline(op, MatvecKind.Forward, m.data, cfg, timings=timings)
    return MatvecResult(BlockVector.time_double(op.dims.n_d, op.dims.n_t, out), t)


def adjoint_matvec(op: SpectralOperator, d: BlockVector, cfg="ddddd", tiling=None,
                   timings: bool = True) -> MatvecResult:
    """matvec.hpp:313-318: m = F* d."""
    if not isinstance(d, BlockVector):
        d = BlockVector.time_double(op.dims.n_d, op.dims.n_t, d)
    _check_input(op, d, False)
    out, t = run_pipeline(op, MatvecKind.Adjoint, d.data, cfg, timings=timings)
    return MatvecResult(BlockVector.time_double(op.dims.n_m, op.dims.n_t, out), t)


def matvec_host_async(op: SpectralOperator, kind: MatvecKind, x, y, cfg="ddddd", ctx: Optional[Context] = None):
    """Queued host-I/O matvec (fmv_matvec_host_async): ``x``
    and ``y`` are PINNED host torch float64 tensors (n_in*nt / n_out*nt);
    the call enqueues the copies and the pipeline and returns at once.
    ``y`` holds the result after ``ctx.synchronize()``; consecutive calls
    overlap each other's copies with their SBGEMVs."""
    ctx = ctx or op.ctx
    fwd = kind == MatvecKind.Forward
    n_in = (op.dims.n_m if fwd else op.dims.n_d) * op.dims.n_t
    n_out = (op.dims.n_d if fwd else op.dims.n_m) * op.dims.n_t
    if x.numel() != n_in or y.numel() != n_out:
        raise ValueError("matvec: input length does not match operator dims")
    check(lib().fmv_matvec_host_async(ctx.handle, op.handle, 0 if fwd else 1, _cfg_str(cfg).encode(),
                                      ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))


def matvec_block(op: SpectralOperator, kind: MatvecKind, inp, cfg="ddddd", ctx: Optional[Context] = None):
    """Block (multi-RHS) matvec: applies F (Forward) or F*
    (Adjoint) to K vectors at once. ``inp`` is (K, n_in*nt) float64 -- a
    numpy array (host I/O) or a CUDA torch tensor (device I/O); returns
    (K, n_out*nt) of the same kind. Row r equals run_pipeline(op, kind,
    inp[r], cfg) up to summation order; the operator is streamed from HBM
    once per 8 right-hand sides."""
    ctx = ctx or op.ctx
    fwd = kind == MatvecKind.Forward
    n_in = (op.dims.n_m if fwd else op.dims.n_d) * op.dims.n_t
    n_out = (op.dims.n_d if fwd else op.dims.n_m) * op.dims.n_t
    cs = _cfg_str(cfg).encode()
    if _is_cuda_tensor(inp):
        import torch

        if inp.dtype != torch.float64 or inp.dim() != 2 or inp.shape[1] != n_in:
            raise ValueError("matvec_block: input must be (K, n_in*n_t) float64")
        x = inp.contiguous()
        out = torch.empty((x.shape[0], n_out), dtype=torch.float64, device=x.device)
        torch.cuda.current_stream(x.device).synchronize()
        check(lib().fmv_matvec_block(ctx.handle, op.handle, int(kind), cs, x.shape[0], ctypes.c_void_p(x.data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()), 1))
        return out
    x = np.ascontiguousarray(inp, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != n_in:
        raise ValueError("matvec_block: input must be (K, n_in*n_t) float64")
    out = np.empty((x.shape[0], n_out), dtype=np.float64)
    check(lib().fmv_matvec_block(ctx.handle, op.handle, int(kind), cs, x.shape[0], x.ctypes.data, out.ctypes.data, 0))
    return out


def forward_matvec_block(op: SpectralOperator, M, cfg="ddddd"):
    """D = F M for K parameter vectors (rows of M, each n_m*n_t, SOTI)."""
    return matvec_block(op, MatvecKind.Forward, M, cfg)


def adjoint_matvec_block(op: SpectralOperator, D, cfg="ddddd"):
    """M = F* D for K sensor vectors (rows of D, each n_d*n_t, SOTI)."""
    return matvec_block(op, MatvecKind.Adjoint, D, cfg)


class MatvecGraph:
    """A device-resident matvec captured once into a CUDA graph
    (fmv_graph_create) and replayed with one cudaGraphLaunch per call on the
    context's stream: ``inp`` / ``out`` are CUDA float64 tensors whose
    contents are read / written at each ``launch()``. For iterative solvers
    applying F / F* many times to the same buffers."""

    def __init__(self, op: SpectralOperator, kind: MatvecKind, inp, out, cfg="ddddd", ctx: Optional[Context] = None):
        import torch

        self.ctx = ctx or op.ctx
        fwd = kind == MatvecKind.Forward
        n_in = (op.dims.n_m if fwd else op.dims.n_d) * op.dims.n_t
        n_out = (op.dims.n_d if fwd else op.dims.n_m) * op.dims.n_t
        for t, n in ((inp, n_in), (out, n_out)):
            if not _is_cuda_tensor(t) or t.dtype != torch.float64 or t.numel() != n or not t.is_contiguous():
                raise ValueError("MatvecGraph: inp / out must be contiguous CUDA float64 tensors of the matvec's sizes")
        self._keep = (op, inp, out)
        torch.cuda.current_stream(inp.device).synchronize()
        h = ctypes.c_void_p()
        check(lib().fmv_graph_create(self.ctx.handle, op.handle, int(kind), _cfg_str(cfg).encode(),
                                     ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.byref(h)))
        self.handle = h

    def launch(self) -> None:
        check(lib().fmv_graph_launch(self.handle))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().fmv_graph_destroy(h)
            except Exception:
                pass
            self.handle = None


def casts_performed() -> int:
    """precision.hpp:27-39 (logical conversion passes on the GPU path)."""
    return int(lib().fmv_casts_performed())


def reset_cast_counter() -> None:
    lib().fmv_reset_cast_counter()


# ---------------------------------------------------------------- fills ----
def seed_stream(seed: int, stream: int) -> int:
    """random_fill.hpp:30-32."""
    return int(lib().fmv_seed_stream(seed, stream))


def uniform_fill(count: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """random_fill.hpp:17-27 (mt19937_64, top 53 bits), bit-identical."""
    out = np.empty(count, dtype=np.float64)
    lib().fmv_uniform_fill(count, seed, lo, hi, out.ctypes.data)
    return out


def non_representable_fill(count: int, seed: int) -> np.ndarray:
    """sweep.hpp:32-46."""
    if count < 1:
        raise ValueError("non_representable_fill: count must be >= 1")
    out = np.empty(count, dtype=np.float64)
    check(lib().fmv_non_representable_fill(count, seed, out.ctypes.data))
    return out


def relative_error(x, ref) -> float:
    """sweep.hpp:49-59."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    ref = np.ascontiguousarray(ref, dtype=np.float64).reshape(-1)
    if x.size != ref.size:
        raise ValueError("relative_error: length mismatch")
    out = ctypes.c_double()
    rc = lib().fmv_relative_error(x.size, x.ctypes.data, ref.ctypes.data, ctypes.byref(out))
    if rc:
        raise ValueError("relative_error: zero-norm reference")
    return out.value
