"""ctypes front-ends for the two CPU oracles (TEST INFRASTRUCTURE ONLY).

* ``Ref``  -- oracle/_ref/libfftmv_ref.so: the reference headers compiled
  verbatim (FFTW API served by MKL DFTI), i.e. the reference itself.
* ``Orc``  -- oracle/liboracle.so: our plain-C restatement (fftmv_oracle.c).

Both expose the same methods so tests can parametrize over them.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_char_p, c_double, c_int, c_size_t, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libfftmv_ref.so")
ORC_PATH = os.path.join(HERE, "liboracle.so")


class _Base:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.L = ctypes.CDLL(path)
        p = self.prefix
        L = self.L
        self._f("seed_stream", c_uint64, [c_uint64, c_uint64])
        self._f("uniform_fill", None, [c_size_t, c_uint64, c_double, c_double, c_void_p])
        self._f("non_representable_fill", c_int, [c_size_t, c_uint64, c_void_p])
        self._f("setup_operator", c_void_p, [c_size_t, c_size_t, c_size_t, c_void_p])
        self._f("op_free", None, [c_void_p])
        self._f("op_bins", None, [c_void_p, c_void_p])
        self._f("dense", c_int, [c_int, c_size_t, c_size_t, c_size_t, c_void_p, c_void_p, c_void_p])
        self._f("fft_forward", c_int, [c_size_t, c_size_t, c_int, c_void_p, c_void_p])
        self._f("fft_inverse", c_int, [c_size_t, c_size_t, c_int, c_void_p, c_void_p])
        self._f("grid_split", c_int, [c_size_t, c_size_t, c_void_p])
        self._f("tree_reduce", c_int, [c_size_t, c_size_t, c_void_p, c_int, c_void_p])
        self._f("last_error", c_char_p, [])
        self._f("relative_error", c_int, [c_size_t, c_void_p, c_void_p, POINTER(c_double)])

    def _f(self, name, res, args):
        f = getattr(self.L, self.prefix + name)
        f.restype = res
        f.argtypes = args
        setattr(self, "_" + name, f)

    def err(self) -> str:
        return self._last_error().decode(errors="replace")

    # ---- fills
    def seed_stream(self, seed, stream):
        return int(self._seed_stream(seed, stream))

    def uniform_fill(self, n, seed, lo=-1.0, hi=1.0):
        o = np.empty(n)
        self._uniform_fill(n, seed, lo, hi, o.ctypes.data)
        return o

    def non_representable_fill(self, n, seed):
        o = np.empty(n)
        if self._non_representable_fill(n, seed, o.ctypes.data):
            raise ValueError(self.err())
        return o

    def relative_error(self, x, r):
        x = np.ascontiguousarray(x, dtype=np.float64)
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = c_double()
        if self._relative_error(x.size, x.ctypes.data, r.ctypes.data, ctypes.byref(out)):
            raise ValueError(self.err())
        return out.value

    # ---- operator
    def setup_operator(self, nm, nd, nt, col):
        col = np.ascontiguousarray(col, dtype=np.float64)
        h = self._setup_operator(nm, nd, nt, col.ctypes.data)
        if not h:
            raise ValueError(self.err())
        return _Op(self, h, nm, nd, nt)

    def dense(self, kind, nm, nd, nt, col, x):
        col = np.ascontiguousarray(col, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((nd if kind == 0 else nm) * nt)
        if self._dense(kind, nm, nd, nt, col.ctypes.data, x.ctypes.data, out.ctypes.data):
            raise ValueError(self.err())
        return out

    def fft_forward(self, L, batch, series, prec=1):
        dt = np.float64 if prec else np.float32
        x = np.ascontiguousarray(series, dtype=dt)
        out = np.empty(batch * (L // 2 + 1), dtype=np.complex128 if prec else np.complex64)
        if self._fft_forward(L, batch, prec, x.ctypes.data, out.ctypes.data):
            raise ValueError(self.err())
        return out

    def fft_inverse(self, L, batch, bins, prec=1):
        ct = np.complex128 if prec else np.complex64
        x = np.ascontiguousarray(bins, dtype=ct)
        out = np.empty(batch * L, dtype=np.float64 if prec else np.float32)
        if self._fft_inverse(L, batch, prec, x.ctypes.data, out.ctypes.data):
            raise ValueError(self.err())
        return out

    def grid_split(self, p, nm):
        r = np.empty(2 * p, dtype=np.uint64)
        if self._grid_split(p, nm, r.ctypes.data):
            raise ValueError(self.err())
        return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(p)]

    def tree_reduce(self, bufs, prec_double: bool):
        b = np.ascontiguousarray(np.stack(bufs), dtype=np.float64)
        out = np.empty(b.shape[1])
        if self._tree_reduce(b.shape[0], b.shape[1], b.ctypes.data, 1 if prec_double else 0, out.ctypes.data):
            raise ValueError(self.err())
        return out


class _Op:
    def __init__(self, owner, h, nm, nd, nt):
        self.o, self.h, self.nm, self.nd, self.nt = owner, h, nm, nd, nt

    def bins(self):
        out = np.empty((self.nt + 1) * self.nd * self.nm, dtype=np.complex128)
        self.o._op_bins(self.h, out.ctypes.data)
        return out

    def matvec(self, kind, cfg, x):
        return self.o.matvec(self, kind, cfg, x)

    def __del__(self):
        try:
            self.o._op_free(self.h)
        except Exception:
            pass


class Ref(_Base):
    """The reference itself (headers compiled verbatim)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_PATH):
        os.environ.setdefault("MKL_NUM_THREADS", "1")
        super().__init__(path)
        self._f("matvec", c_int, [c_void_p, c_int, c_char_p, c_void_p, c_void_p, c_void_p])
        self._f("casts_performed", c_uint64, [])
        self._f("reset_cast_counter", None, [])
        self._f("gemv", c_int, [c_int, c_int, c_char, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, c_void_p,
                                c_size_t, c_size_t, c_void_p, c_size_t, c_size_t, c_void_p, c_size_t, c_size_t,
                                c_size_t, c_double, c_size_t])
        self._f("setup_partitioned", c_void_p, [c_size_t, c_size_t, c_size_t, c_void_p, c_size_t])
        self._f("pop_free", None, [c_void_p])
        self._f("matvec_partitioned", c_int, [c_void_p, c_int, c_char_p, c_void_p, c_void_p, c_void_p])
        self._f("sweep", c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_double, c_void_p, c_void_p])
        self._f("pareto", c_int, [c_size_t, c_void_p, c_void_p, c_char_p, c_void_p])
        self._f("optimal", c_int, [c_size_t, c_void_p, c_void_p, c_char_p, c_double, c_void_p])
        self._f("throughput", c_int, [c_void_p, c_int, c_char_p, c_void_p, c_int, c_int, POINTER(c_double)])
        self._f("throughput_mixed", c_int, [c_void_p, c_char_p, c_void_p, c_void_p, c_int, POINTER(c_double)])
        self._f("op_materialize_single", None, [c_void_p])
        self._f("effective_bandwidth", c_int, [c_size_t, c_size_t, c_size_t, c_size_t, c_double, POINTER(c_double)])
        self._f("select_kernel", c_int, [c_size_t, c_size_t, c_int, c_size_t, c_size_t, c_double, c_size_t])
        self._f("parse_config", c_int, [c_char_p, c_void_p])
        self._f("enumerate_configs", None, [c_void_p])

    def matvec(self, op, kind, cfg, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((op.nd if kind == 0 else op.nm) * op.nt)
        t = np.zeros(6)
        if self._matvec(op.h, kind, cfg.encode(), x.ctypes.data, out.ctypes.data, t.ctypes.data):
            raise ValueError(self.err())
        return out

    def matvec_timed(self, op, kind, cfg, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((op.nd if kind == 0 else op.nm) * op.nt)
        t = np.zeros(6)
        if self._matvec(op.h, kind, cfg.encode(), x.ctypes.data, out.ctypes.data, t.ctypes.data):
            raise ValueError(self.err())
        return out, t

    def matvec_many(self, op, jobs, threads=None):
        """Run [(kind, cfg, x), ...] on a shared operator across host threads
        (the reference's matvecs are reentrant on one operator, SPEC.md:291;
        ctypes drops the GIL for the call). Returns the outputs in job order."""
        from concurrent.futures import ThreadPoolExecutor

        threads = threads or min(len(jobs), len(os.sched_getaffinity(0)))
        with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
            return list(ex.map(lambda j: self.matvec(op, j[0], j[1], j[2]), jobs))

    def throughput(self, op, kind, cfg, x, threads, per_thread):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = c_double()
        if self._throughput(op.h, kind, cfg.encode(), x.ctypes.data, threads, per_thread, ctypes.byref(s)):
            raise RuntimeError(self.err())
        return s.value

    def throughput_mixed(self, op, cfg, m, d, threads):
        m = np.ascontiguousarray(m, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        s = c_double()
        if self._throughput_mixed(op.h, cfg.encode(), m.ctypes.data, d.ctypes.data, threads, ctypes.byref(s)):
            raise RuntimeError(self.err())
        return s.value

    def casts(self):
        return int(self._casts_performed())

    def reset_casts(self):
        self._reset_cast_counter()

    def gemv(self, impl, mode, dtype, m, n, batch, lda, sa, A, sx, x, sy, y, col_tile=256, row_chunk=64,
             ratio=1.0, cutoff=1024):
        rc = self._gemv(impl, mode, dtype.encode(), m, n, batch, lda, sa, A.ctypes.data, A.size, sx, x.ctypes.data,
                        x.size, sy, y.ctypes.data, y.size, col_tile, row_chunk, ratio, cutoff)
        if rc:
            raise ValueError(self.err())
        return y

    def matvec_partitioned(self, nm, nd, nt, col, p, kind, cfg, x):
        col = np.ascontiguousarray(col, dtype=np.float64)
        h = self._setup_partitioned(nm, nd, nt, col.ctypes.data, p)
        if not h:
            raise ValueError(self.err())
        try:
            x = np.ascontiguousarray(x, dtype=np.float64)
            out = np.empty((nd if kind == 0 else nm) * nt)
            if self._matvec_partitioned(h, kind, cfg.encode(), x.ctypes.data, out.ctypes.data, None):
                raise ValueError(self.err())
            return out
        finally:
            self._pop_free(h)

    def sweep(self, op, kind, x, reps, warmup, tol):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows = np.zeros(32 * 4)
        chosen = ctypes.create_string_buffer(6)
        if self._sweep(op.h, kind, x.ctypes.data, reps, warmup, tol, rows.ctypes.data, chosen):
            raise ValueError(self.err())
        return rows.reshape(32, 4), chosen.value.decode()

    def pareto(self, means, errs, cfgs):
        n = len(cfgs)
        m = np.ascontiguousarray(means, dtype=np.float64)
        e = np.ascontiguousarray(errs, dtype=np.float64)
        mask = np.zeros(n, dtype=np.int32)
        if self._pareto(n, m.ctypes.data, e.ctypes.data, "".join(cfgs).encode(), mask.ctypes.data):
            raise ValueError(self.err())
        return mask.astype(bool)

    def optimal(self, means, errs, cfgs, tol):
        n = len(cfgs)
        m = np.ascontiguousarray(means, dtype=np.float64)
        e = np.ascontiguousarray(errs, dtype=np.float64)
        out = ctypes.create_string_buffer(6)
        if self._optimal(n, m.ctypes.data, e.ctypes.data, "".join(cfgs).encode(), tol, out):
            raise ValueError(self.err())
        return out.value.decode()


class Orc(_Base):
    """Plain-C restatement (oracle/fftmv_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = ORC_PATH):
        super().__init__(path)
        self._f("matvec", c_int, [c_void_p, c_int, c_char_p, c_void_p, c_void_p, POINTER(c_uint64)])
        self._f("matvec_partitioned", c_int, [c_size_t, c_size_t, c_size_t, c_void_p, c_size_t, c_int, c_char_p,
                                              c_void_p, c_void_p])
        self._f("gemv", c_int, [c_int, c_char, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, c_void_p, c_size_t,
                                c_void_p, c_size_t, c_void_p])
        self._f("effective_bandwidth", c_int, [c_size_t, c_size_t, c_size_t, c_size_t, c_double, POINTER(c_double)])

    def matvec(self, op, kind, cfg, x, with_casts=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((op.nd if kind == 0 else op.nm) * op.nt)
        c = c_uint64()
        if self._matvec(op.h, kind, cfg.encode(), x.ctypes.data, out.ctypes.data, ctypes.byref(c)):
            raise ValueError(self.err())
        return (out, int(c.value)) if with_casts else out

    def matvec_partitioned(self, nm, nd, nt, col, p, kind, cfg, x):
        col = np.ascontiguousarray(col, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((nd if kind == 0 else nm) * nt)
        if self._matvec_partitioned(nm, nd, nt, col.ctypes.data, p, kind, cfg.encode(), x.ctypes.data,
                                    out.ctypes.data):
            raise ValueError(self.err())
        return out

    def gemv(self, mode, dtype, m, n, batch, lda, sa, A, sx, x, sy, y):
        if self._gemv(mode, dtype.encode(), m, n, batch, lda, sa, A.ctypes.data, sx, x.ctypes.data, sy,
                      y.ctypes.data):
            raise ValueError(self.err())
        return y


_ref = None
_orc = None


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def orc() -> Orc:
    global _orc
    if _orc is None:
        _orc = Orc()
    return _orc


def have_ref() -> bool:
    return os.path.exists(REF_PATH)
