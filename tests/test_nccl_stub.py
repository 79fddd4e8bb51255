"""CPU checks of the host-staged NCCL test transport (tests/stub/fmv_nccl_stub.cpp,
loaded by the library through FMV_NCCL_LIB for multi-process runs on one GPU):
all-gather / broadcast / all-reduce / comm-split semantics at world size 2 and
4 with host buffers, and the timeout error a dead peer produces."""
import ctypes
import os
import subprocess

import numpy as np
import pytest
import multiprocessing as mp

from conftest import ROOT

STUB = os.path.join(ROOT, "build", "libfmv_nccl_stub.so")


class _Id(ctypes.Structure):  # ncclUniqueId is passed by value
    _fields_ = [("internal", ctypes.c_char * 128)]


def _lib():
    if not os.path.exists(STUB):
        subprocess.run(["make", "-C", ROOT, "stub"], check=True, capture_output=True)
    L = ctypes.CDLL(STUB)
    vp = ctypes.c_void_p
    L.ncclGetUniqueId.argtypes = [ctypes.c_char_p]
    L.ncclCommInitRank.argtypes = [ctypes.POINTER(vp), ctypes.c_int, _Id, ctypes.c_int]
    L.ncclAllGather.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_int, vp, vp]
    L.ncclBroadcast.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, vp, vp]
    L.ncclAllReduce.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, vp, vp]
    L.ncclCommSplit.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), vp]
    L.ncclCommGetAsyncError.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    L.ncclCommDestroy.argtypes = [vp]
    return L


def _worker(rank, world, idb, q):
    os.environ["FMV_STUB_TIMEOUT_S"] = "3"
    L = _lib()
    comm = ctypes.c_void_p()
    assert L.ncclCommInitRank(ctypes.byref(comm), world, _Id.from_buffer_copy(idb), rank) == 0
    n = 300_000  # > one 2 MiB staging slot in doubles: exercises the chunk loop
    mine = np.arange(n, dtype=np.float64) * (rank + 1)
    gath = np.empty(world * n)
    assert L.ncclAllGather(mine.ctypes.data, gath.ctypes.data, n, 8, comm, None) == 0
    b = np.full(1000, -1.0, dtype=np.float32)
    if rank == world - 1:
        b[:] = np.arange(1000, dtype=np.float32)
    assert L.ncclBroadcast(b.ctypes.data, b.ctypes.data, 1000, 7, world - 1, comm, None) == 0
    red = np.empty(n)
    assert L.ncclAllReduce(mine.ctypes.data, red.ctypes.data, n, 8, 0, comm, None) == 0
    # 2-D style split: color = rank // 2 (rows), key = rank % 2
    sub = ctypes.c_void_p()
    assert L.ncclCommSplit(comm, rank // 2, rank % 2, ctypes.byref(sub), None) == 0
    s_in = np.array([float(rank)])
    s_out = np.empty(2)
    assert L.ncclAllGather(s_in.ctypes.data, s_out.ctypes.data, 1, 8, sub, None) == 0
    L.ncclCommDestroy(sub)
    # a peer that never arrives: rank 0 waits alone and times out
    err = ctypes.c_int(0)
    rc = 0
    if rank == 0:
        rc = L.ncclAllGather(mine.ctypes.data, gath.ctypes.data, 1, 8, comm, None)
        L.ncclCommGetAsyncError(comm, ctypes.byref(err))
    q.put((rank, gath, b, red, s_out, rc, err.value))


@pytest.mark.parametrize("world", [2, 4])
def test_stub_collectives(world):
    L = _lib()
    idb = ctypes.create_string_buffer(128)
    assert L.ncclGetUniqueId(idb) == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, bytes(idb.raw), q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    n = 300_000
    base = np.arange(n, dtype=np.float64)
    want_g = np.concatenate([base * (r + 1) for r in range(world)])
    want_r = sum(base * (r + 1) for r in range(world))
    for rank, gath, b, red, s_out, rc, err in res:
        assert np.array_equal(gath, want_g)
        assert np.array_equal(b, np.arange(1000, dtype=np.float32))
        assert np.array_equal(red, want_r)
        assert list(s_out) == [2 * (rank // 2), 2 * (rank // 2) + 1]
        if rank == 0:
            assert rc == 6 and err == 6  # ncclRemoteError after FMV_STUB_TIMEOUT_S
