"""1 x p column partition of the operator (partition.hpp:19-238).

Two execution modes:

* In-process (reference semantics, partition.hpp:1-8): every shard is its
  own SpectralOperator on one GPU, shards run one after another and the
  forward partials meet in the reference's fixed left-balanced tree in cfg[4]
  precision. Used for parity with the reference's simulated partition.
* Distributed (the B200 deployment): one process per GPU. Each rank holds
  its shard's operator; the forward partial d is summed with an NCCL
  all-reduce in cfg[4] precision and the adjoint input is broadcast in cfg[0]
  precision, both issued from inside libfftmv_cuda (fmv_matvec_partitioned)
  on the matvec's own stream. A torch.distributed transport (gloo on CPU,
  nccl on GPU) with an injectable per-shard compute covers the same host
  logic in CPU tests.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _capi
from ._capi import check, lib
from .fftmv import (BlockColumn, BlockVector, Context, Domain, Layout, MatvecKind, PhaseTimings, Precision,
                    PrecisionConfig, ProblemDims, SpectralOperator, _cfg_str, _is_cuda_tensor, default_context,
                    run_pipeline, setup_operator)

__all__ = ["Grid1xP", "CommSpec", "shard_operator", "tree_reduce", "PartitionedOperator", "PartitionedResult",
           "setup_partitioned", "forward_matvec_partitioned", "adjoint_matvec_partitioned", "round_to",
           "DistributedMatvec", "GridPxQ", "shard_operator_2d", "PartitionedOperator2D", "setup_partitioned_2d",
           "forward_matvec_partitioned_2d", "adjoint_matvec_partitioned_2d", "DistributedMatvec2D"]


@dataclass
class Grid1xP:
    """partition.hpp:23-43: balanced contiguous Nm ranges, leading ranges take the remainder."""

    p: int = 1
    shard_ranges: List[tuple] = field(default_factory=list)

    @staticmethod
    def split(p: int, n_m: int) -> "Grid1xP":
        if p < 1:
            raise ValueError("Grid1xP: p must be >= 1")
        if p > n_m:
            raise ValueError("Grid1xP: more workers than parameter columns")
        base, rem = divmod(n_m, p)
        ranges, begin = [], 0
        for w in range(p):
            size = base + (1 if w < rem else 0)
            ranges.append((begin, begin + size))
            begin += size
        return Grid1xP(p, ranges)

    def shard_size(self, w: int) -> int:
        return self.shard_ranges[w][1] - self.shard_ranges[w][0]


@dataclass
class CommSpec:
    """partition.hpp:47-59: both collectives move n_d * n_t values."""

    class Op(enum.IntEnum):
        Reduce = 0
        Broadcast = 1

    op: "CommSpec.Op"
    precision: Precision
    buffer_len: int

    @staticmethod
    def forward_reduce(cfg: PrecisionConfig, dims: ProblemDims) -> "CommSpec":
        return CommSpec(CommSpec.Op.Reduce, cfg[4], dims.n_d * dims.n_t)

    @staticmethod
    def adjoint_broadcast(cfg: PrecisionConfig, dims: ProblemDims) -> "CommSpec":
        return CommSpec(CommSpec.Op.Broadcast, cfg[0], dims.n_d * dims.n_t)


def shard_operator(col: BlockColumn, grid: Grid1xP) -> List[BlockColumn]:
    """partition.hpp:63-80: worker w gets columns [lo, hi) of every block."""
    d = col.dims
    if not grid.shard_ranges or grid.shard_ranges[-1][1] != d.n_m:
        raise ValueError("shard_operator: grid does not cover n_m")
    blocks = np.asarray(col.data).reshape(d.n_t, d.n_m, d.n_d)  # [t][j][i] (column-major blocks)
    out = []
    for lo, hi in grid.shard_ranges:
        out.append(BlockColumn(ProblemDims(hi - lo, d.n_d, d.n_t), np.ascontiguousarray(blocks[:, lo:hi, :]).reshape(-1)))
    return out


def round_to(x: np.ndarray, p: str) -> np.ndarray:
    """Value rounding to a phase precision (precision.hpp:44-61; 'h' = fp16 ext.)."""
    if p == "s":
        return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
    if p == "h":
        return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)
    return np.asarray(x, dtype=np.float64)


def tree_reduce(buffers: List[np.ndarray], precision: Precision) -> np.ndarray:
    """partition.hpp:84-132: inputs cast to `precision`, fixed left-balanced
    pairwise tree ((b0+b1)+(b2+b3)), ((b0+b1)+b2) for odd counts, root -> double."""
    if not buffers:
        raise ValueError("tree_reduce: no buffers")
    n = len(buffers[0])
    dt = np.float64 if precision == Precision.Double else np.float32
    level = []
    for b in buffers:
        if len(b) != n:
            raise ValueError("tree_reduce: buffer length mismatch")
        level.append(np.asarray(b, dtype=np.float64).astype(dt))
    while len(level) > 1:
        nxt = [level[k] + level[k + 1] for k in range(0, len(level) - 1, 2)]
        if len(level) % 2 == 1:
            nxt.append(level[-1])
        level = nxt
    return level[0].astype(np.float64)


# ---------------------------------------------------- in-process (simulated) ---
@dataclass
class PartitionedOperator:
    """partition.hpp:135-147."""

    dims: ProblemDims
    grid: Grid1xP
    workers: List[SpectralOperator]


@dataclass
class PartitionedResult:
    output: BlockVector
    timings: PhaseTimings


def setup_partitioned(col: BlockColumn, grid: Grid1xP, ctx: Optional[Context] = None) -> PartitionedOperator:
    return PartitionedOperator(col.dims, grid, [setup_operator(s, ctx) for s in shard_operator(col, grid)])


def _payload_cfg(cfg: str) -> str:
    # The broadcast payload is already rounded to cfg[0] (partition.hpp:198-203);
    # padding it again is exact, so the shard pipeline runs with slot 0 = 'd'.
    return "d" + cfg[1:]


def forward_matvec_partitioned(pop: PartitionedOperator, m, cfg="ddddd") -> PartitionedResult:
    """partition.hpp:157-182 (restated: the reference's own check at :159
    rejects every p >= 2)."""
    c = _cfg_str(cfg)
    m = np.ascontiguousarray(m.data if isinstance(m, BlockVector) else m, dtype=np.float64).reshape(-1)
    nt = pop.dims.n_t
    if m.size != pop.dims.n_m * nt:
        raise ValueError("partitioned matvec: input extents do not match dims")
    total = PhaseTimings()
    partials = []
    for (lo, hi), op in zip(pop.grid.shard_ranges, pop.workers):
        part, t = run_pipeline(op, MatvecKind.Forward, m[lo * nt:hi * nt], c)
        total += t
        partials.append(part)
    d = tree_reduce(partials, Precision.Double if c[4] == "d" else Precision.Single)
    return PartitionedResult(BlockVector.time_double(pop.dims.n_d, nt, d), total)


def adjoint_matvec_partitioned(pop: PartitionedOperator, d, cfg="ddddd") -> PartitionedResult:
    """partition.hpp:187-217: cast d to cfg[0] once, every shard pads from that payload."""
    c = _cfg_str(cfg)
    d = np.ascontiguousarray(d.data if isinstance(d, BlockVector) else d, dtype=np.float64).reshape(-1)
    nt = pop.dims.n_t
    if d.size != pop.dims.n_d * nt:
        raise ValueError("partitioned matvec: input extents do not match dims")
    payload = round_to(d, c[0])  # one cast (partition.hpp:198-203), stored in cfg[0]'s own type
    total = PhaseTimings()
    out = np.empty(pop.dims.n_m * nt)
    for (lo, hi), op in zip(pop.grid.shard_ranges, pop.workers):
        shard, t = run_pipeline(op, MatvecKind.Adjoint, payload, c, payload=c[0])
        total += t
        out[lo * nt:hi * nt] = shard
    return PartitionedResult(BlockVector.time_double(pop.dims.n_m, nt, out), total)


# ------------------------------------------------------------ distributed ---
class DistributedMatvec:
    """One rank of a 1 x p partitioned operator.

    transport="native": NCCL inside libfftmv_cuda (fmv_comm_init +
      fmv_matvec_partitioned); requires torch.distributed to be initialised
      (used only to ship rank 0's NCCL unique id).
    transport="torch": collectives through torch.distributed (gloo or nccl)
      on host arrays, compute through ``compute(kind, cfg, x) -> np.ndarray``
      (default: this rank's GPU shard via run_pipeline). Lets the host logic
      run with world_size > 1 on CPU.
    """

    def __init__(self, dims: ProblemDims, rank: int, world: int, shard: Optional[SpectralOperator] = None,
                 transport: str = "native", compute: Optional[Callable] = None, ctx: Optional[Context] = None):
        self.dims = dims
        self.rank = rank
        self.world = world
        self.grid = Grid1xP.split(world, dims.n_m)
        self.lo, self.hi = self.grid.shard_ranges[rank]
        self.shard = shard
        self.transport = transport
        self.ctx = ctx or (shard.ctx if shard is not None else None)
        if transport == "native":
            if shard is None:
                raise ValueError("native transport needs the rank's SpectralOperator shard")
            self._init_native()
        elif transport == "torch":
            self.compute = compute or (lambda kind, cfg, x: run_pipeline(self.shard, kind, x, cfg)[0])
        else:
            raise ValueError("transport must be 'native' or 'torch'")

    def _init_native(self):
        import torch.distributed as dist

        # rank 0's NCCL id, shipped with torch.distributed (a 1-rank run still
        # builds a real 1-rank communicator, so the collectives execute)
        idb = (ctypes.c_char * 128)()
        if self.rank == 0:
            check(lib().fmv_comm_unique_id(idb))
        if self.world > 1:
            obj = [bytes(idb)] if self.rank == 0 else [None]
            dist.broadcast_object_list(obj, src=0)
            idb = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        check(lib().fmv_comm_init(self.ctx.handle, self.world, self.rank, idb))

    # -- forward: local slice in, full d out on every rank
    def forward(self, m_slice, cfg="ddddd", times: bool = False):
        c = _cfg_str(cfg)
        nt = self.dims.n_t
        if self.transport == "native":
            return self._native(MatvecKind.Forward, c, m_slice, self.dims.n_d * nt, times)
        import torch
        import torch.distributed as dist

        part = np.asarray(self.compute(MatvecKind.Forward, c, np.ascontiguousarray(m_slice, dtype=np.float64)))
        if self.world == 1:
            return part
        t = torch.from_numpy(part.astype(np.float64 if c[4] == "d" else np.float32))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy().astype(np.float64)

    # -- adjoint: full d (rank 0) in, local m slice out
    def adjoint(self, d_full, cfg="ddddd", times: bool = False):
        c = _cfg_str(cfg)
        nt = self.dims.n_t
        n_slice = (self.hi - self.lo) * nt
        if self.transport == "native":
            return self._native(MatvecKind.Adjoint, c, d_full, n_slice, times)
        import torch
        import torch.distributed as dist

        nd = self.dims.n_d * nt
        bdt = {"d": np.float64, "s": np.float32, "h": np.float16}[c[0]]
        buf = np.zeros(nd, dtype=bdt)
        if self.rank == 0:
            buf[:] = np.asarray(d_full, dtype=np.float64).astype(bdt)
        t = torch.from_numpy(buf)
        if self.world > 1:
            dist.broadcast(t, src=0)
        payload = t.numpy().astype(np.float64)
        return np.asarray(self.compute(MatvecKind.Adjoint, _payload_cfg(c), payload))

    def _native(self, kind, c, x, n_out, times):
        t = _capi.PhaseTimesC()
        if _is_cuda_tensor(x):
            import torch

            out = torch.empty(n_out, dtype=torch.float64, device=x.device)
            torch.cuda.current_stream(x.device).synchronize()
            check(lib().fmv_matvec_partitioned(self.ctx.handle, self.shard.handle, int(kind), c.encode(),
                                               ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), 1,
                                               ctypes.byref(t) if times else None))
        else:
            out = np.empty(n_out)
            xin = None if x is None else np.ascontiguousarray(x, dtype=np.float64)
            check(lib().fmv_matvec_partitioned(self.ctx.handle, self.shard.handle, int(kind), c.encode(),
                                               None if xin is None else xin.ctypes.data, out.ctypes.data, 0,
                                               ctypes.byref(t) if times else None))
        if times:
            return out, PhaseTimings(list(t.phase_s), t.total_s)
        return out

    def comm_size(self) -> tuple:
        """(nranks, rank) of the library's live communicator (native transport)."""
        n, r = ctypes.c_int(), ctypes.c_int()
        check(lib().fmv_comm_size(self.ctx.handle, ctypes.byref(n), ctypes.byref(r)))
        return n.value, r.value

    def close(self):
        if self.transport == "native" and self.ctx is not None:
            lib().fmv_comm_destroy(self.ctx.handle)


# ================================================================ 2-D grid ===
# SURVEY.md §8 f3 / PAPER.md:341: the 1D column partition generalised to a
# pr x pc grid that splits the sensor rows (Nd) as well as the parameter
# columns (Nm). Rank r sits at grid position (ri, cj) = divmod(r, pc) and
# holds block (ri, cj) of every time block. F: m_cj is broadcast down grid
# column cj (in cfg[0], the pad precision: the payload semantics of the 1 x p
# adjoint, partition.hpp:196-206), every rank computes its partial d_ri, and
# the pc partials of grid row ri are summed in cfg[4] (partition.hpp:175-177).
# F* is the mirror image: d_ri broadcast along the row, partial m_cj summed
# down the column. pr = 1 is exactly the 1 x p partition.


def _balanced(p: int, n: int, what: str) -> List[tuple]:
    if p < 1:
        raise ValueError(f"GridPxQ: {what} must be >= 1")
    if p > n:
        raise ValueError(f"GridPxQ: more {what} than extent {n}")
    base, rem = divmod(n, p)
    out, b = [], 0
    for w in range(p):
        sz = base + (1 if w < rem else 0)
        out.append((b, b + sz))
        b += sz
    return out


@dataclass
class GridPxQ:
    """pr x pc grid: row ranges over Nd, column ranges over Nm (both split
    like Grid1xP::split, partition.hpp:27-40); rank = ri * pc + cj."""

    pr: int = 1
    pc: int = 1
    row_ranges: List[tuple] = field(default_factory=list)
    col_ranges: List[tuple] = field(default_factory=list)

    @staticmethod
    def split(pr: int, pc: int, n_d: int, n_m: int) -> "GridPxQ":
        return GridPxQ(pr, pc, _balanced(pr, n_d, "grid rows"), _balanced(pc, n_m, "grid columns"))

    @property
    def size(self) -> int:
        return self.pr * self.pc

    def coords(self, rank: int) -> tuple:
        if not 0 <= rank < self.size:
            raise ValueError("GridPxQ: rank out of range")
        return divmod(rank, self.pc)


def shard_operator_2d(col: BlockColumn, grid: GridPxQ) -> List[BlockColumn]:
    """Block (ri, cj) of every time block, in rank order (ri * pc + cj)."""
    d = col.dims
    if grid.row_ranges[-1][1] != d.n_d or grid.col_ranges[-1][1] != d.n_m:
        raise ValueError("shard_operator_2d: grid does not cover (n_d, n_m)")
    blocks = np.asarray(col.data).reshape(d.n_t, d.n_m, d.n_d)  # [t][j][i]
    out = []
    for dlo, dhi in grid.row_ranges:
        for mlo, mhi in grid.col_ranges:
            sub = np.ascontiguousarray(blocks[:, mlo:mhi, dlo:dhi]).reshape(-1)
            out.append(BlockColumn(ProblemDims(mhi - mlo, dhi - dlo, d.n_t), sub))
    return out


@dataclass
class PartitionedOperator2D:
    dims: ProblemDims
    grid: GridPxQ
    workers: List[SpectralOperator]  # rank order


def setup_partitioned_2d(col: BlockColumn, grid: GridPxQ, ctx: Optional[Context] = None) -> PartitionedOperator2D:
    return PartitionedOperator2D(col.dims, grid, [setup_operator(s, ctx) for s in shard_operator_2d(col, grid)])


def _matvec_2d(pop: PartitionedOperator2D, x, cfg, fwd: bool, compute=None) -> PartitionedResult:
    c = _cfg_str(cfg)
    nt = pop.dims.n_t
    g = pop.grid
    x = np.ascontiguousarray(x.data if isinstance(x, BlockVector) else x, dtype=np.float64).reshape(-1)
    if x.size != (pop.dims.n_m if fwd else pop.dims.n_d) * nt:
        raise ValueError("partitioned matvec: input extents do not match dims")
    kind = MatvecKind.Forward if fwd else MatvecKind.Adjoint
    run = compute or (lambda r, k, cc, v: run_pipeline(pop.workers[r], k, v, cc)[0])
    in_ranges, out_ranges = (g.col_ranges, g.row_ranges) if fwd else (g.row_ranges, g.col_ranges)
    payloads = [round_to(x[lo * nt:hi * nt], c[0]) for lo, hi in in_ranges]  # broadcast once per input slice
    out = np.empty((pop.dims.n_d if fwd else pop.dims.n_m) * nt)
    for o, (lo, hi) in enumerate(out_ranges):
        partials = []
        for i in range(len(in_ranges)):
            r = o * g.pc + i if fwd else i * g.pc + o
            partials.append(np.asarray(run(r, kind, _payload_cfg(c), payloads[i])))
        out[lo * nt:hi * nt] = tree_reduce(partials, Precision.Double if c[4] == "d" else Precision.Single) \
            if len(partials) > 1 else partials[0]
    return PartitionedResult(BlockVector.time_double(pop.dims.n_d if fwd else pop.dims.n_m, nt, out), PhaseTimings())


def forward_matvec_partitioned_2d(pop: PartitionedOperator2D, m, cfg="ddddd") -> PartitionedResult:
    """d = F m on the pr x pc grid, simulated in process (one GPU, shards in
    rank order, row sums in the fixed tree_reduce order)."""
    return _matvec_2d(pop, m, cfg, True)


def adjoint_matvec_partitioned_2d(pop: PartitionedOperator2D, d, cfg="ddddd") -> PartitionedResult:
    """m = F* d on the pr x pc grid, simulated in process."""
    return _matvec_2d(pop, d, cfg, False)


class DistributedMatvec2D:
    """One rank of a pr x pc grid (rank = ri * pc + cj).

    transport="native": NCCL row/column communicators inside libfftmv_cuda
      (fmv_comm_init_2d, ncclCommSplit) and fmv_matvec_partitioned_2d.
    transport="torch": torch.distributed row/column groups (gloo or nccl) on
      host arrays with an injectable ``compute(kind, cfg, x)`` -- the CPU
      tests of the orchestration.
    forward(m_cj) -> d_ri (m_cj needed on grid row 0 only); adjoint(d_ri) ->
    m_cj (d_ri needed on grid column 0 only).
    """

    def __init__(self, dims: ProblemDims, pr: int, pc: int, rank: int, shard: Optional[SpectralOperator] = None,
                 transport: str = "native", compute: Optional[Callable] = None, ctx: Optional[Context] = None):
        self.dims = dims
        self.grid = GridPxQ.split(pr, pc, dims.n_d, dims.n_m)
        self.rank = rank
        self.ri, self.cj = self.grid.coords(rank)
        self.dlo, self.dhi = self.grid.row_ranges[self.ri]
        self.mlo, self.mhi = self.grid.col_ranges[self.cj]
        self.shard = shard
        self.transport = transport
        self.ctx = ctx or (shard.ctx if shard is not None else None)
        if transport == "native":
            if shard is None:
                raise ValueError("native transport needs the rank's SpectralOperator shard")
            import torch.distributed as dist

            idb = (ctypes.c_char * 128)()
            if rank == 0:
                check(lib().fmv_comm_unique_id(idb))
            if self.grid.size > 1:
                obj = [bytes(idb)] if rank == 0 else [None]
                dist.broadcast_object_list(obj, src=0)
                idb = (ctypes.c_char * 128).from_buffer_copy(obj[0])
            check(lib().fmv_comm_init_2d(self.ctx.handle, pr, pc, rank, idb))
        elif transport == "torch":
            import torch.distributed as dist

            self.compute = compute or (lambda kind, cfg, x: run_pipeline(self.shard, kind, x, cfg)[0])
            # every rank creates every group in the same order (torch.distributed requirement)
            self.rows = [dist.new_group([i * pc + j for j in range(pc)]) if pr * pc > 1 else None for i in range(pr)]
            self.cols = [dist.new_group([i * pc + j for i in range(pr)]) if pr * pc > 1 else None for j in range(pc)]
        else:
            raise ValueError("transport must be 'native' or 'torch'")

    def _torch(self, kind, c, x, bgroup, broot, bsize, rgroup, rsize, n_in):
        import torch
        import torch.distributed as dist

        bdt = {"d": np.float64, "s": np.float32, "h": np.float16}[c[0]]
        buf = np.zeros(n_in, dtype=bdt)
        if x is not None:
            buf[:] = np.asarray(x, dtype=np.float64).astype(bdt)
        t = torch.from_numpy(buf)
        if bsize > 1:
            dist.broadcast(t, src=broot, group=bgroup)
        part = np.asarray(self.compute(kind, _payload_cfg(c), t.numpy().astype(np.float64)))
        if rsize == 1:
            return part
        r = torch.from_numpy(part.astype(np.float64 if c[4] == "d" else np.float32))
        dist.all_reduce(r, op=dist.ReduceOp.SUM, group=rgroup)
        return r.numpy().astype(np.float64)

    def forward(self, m_slice, cfg="ddddd"):
        c = _cfg_str(cfg)
        nt = self.dims.n_t
        g = self.grid
        if self.transport == "native":
            return self._native(MatvecKind.Forward, c, m_slice, (self.dhi - self.dlo) * nt)
        return self._torch(MatvecKind.Forward, c, m_slice if self.ri == 0 else None, self.cols[self.cj], self.cj, g.pr,
                           self.rows[self.ri], g.pc, (self.mhi - self.mlo) * nt)

    def adjoint(self, d_slice, cfg="ddddd"):
        c = _cfg_str(cfg)
        nt = self.dims.n_t
        g = self.grid
        if self.transport == "native":
            return self._native(MatvecKind.Adjoint, c, d_slice, (self.mhi - self.mlo) * nt)
        return self._torch(MatvecKind.Adjoint, c, d_slice if self.cj == 0 else None, self.rows[self.ri],
                           self.ri * g.pc, g.pc, self.cols[self.cj], g.pr, (self.dhi - self.dlo) * nt)

    def _native(self, kind, c, x, n_out):
        if _is_cuda_tensor(x):
            import torch

            out = torch.empty(n_out, dtype=torch.float64, device=x.device)
            torch.cuda.current_stream(x.device).synchronize()
            check(lib().fmv_matvec_partitioned_2d(self.ctx.handle, self.shard.handle, int(kind), c.encode(),
                                                  ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), 1))
            return out
        out = np.empty(n_out)
        xin = None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        check(lib().fmv_matvec_partitioned_2d(self.ctx.handle, self.shard.handle, int(kind), c.encode(),
                                              None if xin is None else xin.ctypes.data, out.ctypes.data, 0))
        return out

    def close(self):
        if self.transport == "native" and self.ctx is not None:
            lib().fmv_comm_destroy(self.ctx.handle)
