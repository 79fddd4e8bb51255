"""Queued host-I/O matvecs (fmv_matvec_host_async, an addition to the
reference's blocking run_pipeline, matvec.hpp:233-289): several F / F* calls
with pinned host buffers enqueued back to back, one fmv_synchronize, and every
result equal bit for bit to the same pipeline run another way -- the
device-resident fmv_matvec_async (queued calls are unchunked by default), or,
with FMV_QCHUNKS = FMV_CHUNKS = c, the blocking fmv_matvec on the same pinned
buffers (same column-chunk plan) -- and pinned to the reference golden
outputs. Run with -m gpu."""
import ctypes

import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import configs32, golden, make_inputs, rel
from paper_2508_10202_b200 import _capi

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


def _queue_vs_blocking(op, ctx, calls, cfg, against="device"):
    """calls: [(kind, x)] -- queue them all, then compare each with the
    device-resident call (against="device") or the blocking call on the same
    pinned buffers (against="blocking")."""
    import torch

    L = F.lib()
    nm, nd, nt = op.dims.n_m, op.dims.n_d, op.dims.n_t
    ins = [_pinned(x) for _, x in calls]
    outs = [torch.full(((nd if k == 0 else nm) * nt,), np.nan, dtype=torch.float64).pin_memory() for k, _ in calls]
    for (k, _), xi, yo in zip(calls, ins, outs):
        _capi.check(L.fmv_matvec_host_async(ctx.handle, op.handle, k, cfg.encode(), ctypes.c_void_p(xi.data_ptr()),
                                            ctypes.c_void_p(yo.data_ptr())))
    ctx.synchronize()
    got = [y.numpy().copy() for y in outs]
    want = []
    for (k, _), xi, yo in zip(calls, ins, outs):
        if against == "blocking":
            _capi.check(L.fmv_matvec(ctx.handle, op.handle, k, cfg.encode(), ctypes.c_void_p(xi.data_ptr()),
                                     ctypes.c_void_p(yo.data_ptr()), 0, None))
            want.append(yo.numpy().copy())
        else:
            dx, dy = xi.cuda(), torch.empty(yo.numel(), dtype=torch.float64, device="cuda")
            _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, k, cfg.encode(), ctypes.c_void_p(dx.data_ptr()),
                                           ctypes.c_void_p(dy.data_ptr())))
            ctx.synchronize()
            want.append(dy.cpu().numpy())
    for i, (g, w) in enumerate(zip(got, want)):
        assert np.array_equal(g, w), (cfg, i, calls[i][0], rel(g, w))
    return got


@pytest.mark.parametrize("chunks", [None, "3", "6"])
def test_queued_equals_blocking_and_golden_C1(monkeypatch, chunks):
    """C1 (the golden shape), all 32 {d,s} configs: F, F*, F, F*, F*, F with
    fresh inputs per call, queued; equal bitwise to the device-resident calls
    (default, unchunked) or to the blocking calls with the same chunk plan,
    and to the reference golden outputs within each config's tolerance."""
    if chunks:
        monkeypatch.setenv("FMV_CHUNKS", chunks)
        monkeypatch.setenv("FMV_QCHUNKS", chunks)
    g = golden("matvec")
    nm, nd, nt = 100, 10, 100
    col, m, d = make_inputs(F, nm, nd, nt)
    ctx = F.Context(0)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col), ctx)
    rf, ra = g["uni_C1_F_ddddd"], g["uni_C1_A_ddddd"]
    errs = g["uni_C1_errors"]
    rng = np.random.default_rng(7)
    for i, cfg in enumerate(configs32()):
        calls = [(0, m), (1, d), (0, rng.uniform(-1, 1, nm * nt)), (1, rng.uniform(-1, 1, nd * nt)),
                 (1, d), (0, m)]
        got = _queue_vs_blocking(op, ctx, calls, cfg, "blocking" if chunks else "device")
        for j in (0, 5):
            assert rel(got[j], rf) <= max(2 * errs[i, 0], 1e-12), (cfg, j)
        assert rel(got[1], ra) <= max(2 * errs[i, 1], 1e-12), cfg
        assert rel(got[4], ra) <= max(2 * errs[i, 1], 1e-12), cfg


@pytest.mark.parametrize("nt,chunks", [(343, None), (1000, None), (1000, "4")])
def test_queued_medium_many_calls(monkeypatch, nt, chunks):
    """A 0.9 GB operator (queued unchunked, or 4 column chunks like the blocking
    call) and a runtime-plan length (Nt = 343, runtime register FFTs on both
    slots): 10 queued calls with distinct inputs equal the device-resident /
    blocking ones bitwise; fp64 results match the CPU oracle."""
    from oracle.oracle import have_ref, orc, ref

    if chunks:
        monkeypatch.setenv("FMV_QCHUNKS", chunks)
        monkeypatch.setenv("FMV_CHUNKS", chunks)
    nm, nd = (1200, 48) if nt == 1000 else (600, 24)
    col, m, d = make_inputs(F, nm, nd, nt)
    ctx = F.Context(0)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col), ctx)
    rng = np.random.default_rng(11)
    calls = []
    for i in range(10):
        k = i % 2 if i < 6 else (i // 2) % 2
        calls.append((k, rng.uniform(-1, 1, (nm if k == 0 else nd) * nt)))
    for cfg in ("ddddd", "dssdd"):
        got = _queue_vs_blocking(op, ctx, calls, cfg, "blocking" if chunks else "device")
        if cfg == "ddddd":
            chk = ref() if have_ref() else orc()
            cop = chk.setup_operator(nm, nd, nt, col)
            for (k, x), y in list(zip(calls, got))[:3]:
                assert rel(y, chk.matvec(cop, k, "ddddd", x)) <= 1e-12


def test_queued_rejects_pageable_and_interleaves_with_blocking():
    """Pageable buffers are refused (FMV_EINVAL); queued calls interleaved with
    device-resident async and blocking calls on the same ctx give the same
    results as running each alone."""
    import torch

    L = F.lib()
    nm, nd, nt = 200, 12, 100
    col, m, d = make_inputs(F, nm, nd, nt)
    ctx = F.Context(0)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col), ctx)
    out = np.zeros(nd * nt)
    rc = L.fmv_matvec_host_async(ctx.handle, op.handle, 0, b"ddddd", ctypes.c_void_p(m.ctypes.data),
                                 ctypes.c_void_p(out.ctypes.data))
    assert rc == 1 and b"pinned" in L.fmv_last_error()
    want_f = F.forward_matvec(op, m, "ddddd").output.data
    want_a = F.adjoint_matvec(op, d, "ddddd").output.data
    mp, dp = _pinned(m), _pinned(d)
    yo = [torch.empty(nd * nt, dtype=torch.float64).pin_memory() for _ in range(3)]
    zo = [torch.empty(nm * nt, dtype=torch.float64).pin_memory() for _ in range(3)]
    dd = torch.from_numpy(d).cuda()
    dz = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
    for i in range(3):
        _capi.check(L.fmv_matvec_host_async(ctx.handle, op.handle, 0, b"ddddd", ctypes.c_void_p(mp.data_ptr()),
                                            ctypes.c_void_p(yo[i].data_ptr())))
        _capi.check(L.fmv_matvec_async(ctx.handle, op.handle, 1, b"ddddd", ctypes.c_void_p(dd.data_ptr()),
                                       ctypes.c_void_p(dz.data_ptr())))
        _capi.check(L.fmv_matvec_host_async(ctx.handle, op.handle, 1, b"ddddd", ctypes.c_void_p(dp.data_ptr()),
                                            ctypes.c_void_p(zo[i].data_ptr())))
    _capi.check(L.fmv_join(ctx.handle))
    ctx.synchronize()
    yp = torch.empty(nd * nt, dtype=torch.float64).pin_memory()  # the Python wrapper
    F.matvec_host_async(op, F.MatvecKind.Forward, mp, yp, "ddddd", ctx)
    ctx.synchronize()
    assert np.array_equal(yp.numpy(), want_f)
    with pytest.raises(ValueError):
        F.matvec_host_async(op, F.MatvecKind.Forward, dp, yp, "ddddd", ctx)
    for i in range(3):
        assert np.array_equal(yo[i].numpy(), want_f)
        assert np.array_equal(zo[i].numpy(), want_a)
    assert np.array_equal(dz.cpu().numpy(), want_a)
