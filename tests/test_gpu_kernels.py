"""GPU checks of the L1 kernels through the C ABI: the batched real FFTs
against the SPEC contract and the reference's FFT outputs, and the
strided-batched GEMV against the reference's naive kernel. Run with -m gpu."""
import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import golden, rel

pytestmark = pytest.mark.gpu

D, S = F.Precision.Double, F.Precision.Single


def plan(L, b, p=D, inv=False):
    return F.FftPlan(L, b, p, F.FftDirection.Inverse if inv else F.FftDirection.Forward)


def test_fft_known_answers_and_reference_golden():
    g = golden("fft")
    X = F.forward_real_batched(plan(8, 1), np.ones(8))
    assert abs(X[0] - 8) < 1e-14 and np.allclose(X[1:], 0, atol=1e-14)
    d = np.zeros(8)
    d[0] = 1
    assert np.allclose(F.forward_real_batched(plan(8, 1), d), 1, atol=1e-15)
    x = g["rand16_in"]
    naive = np.array([np.sum(x * np.exp(-2j * np.pi * k * np.arange(16) / 16)) for k in range(9)])
    assert rel(F.forward_real_batched(plan(16, 1), x), naive) < 1e-12
    assert rel(F.forward_real_batched(plan(400, 3), g["rand400x3_in"]), g["rand400x3"]) < 1e-13
    assert rel(F.forward_real_batched(plan(2000, 2), g["rand2000x2_in"]), g["rand2000x2"]) < 1e-13
    assert rel(F.forward_real_batched(plan(400, 3, S), g["rand400x3_in"].astype(np.float32)), g["rand400x3_f32"]) < 1e-5
    assert rel(F.inverse_real_batched(plan(400, 3, inv=True), g["rand400x3"]), g["inv400x3"]) < 1e-13
    assert rel(F.inverse_real_batched(plan(400, 3, S, inv=True), g["rand400x3_f32"]), g["inv400x3_f32"]) < 1e-5
    ones = np.zeros(5, dtype=complex)
    ones[0] = 8
    assert np.allclose(F.inverse_real_batched(plan(8, 1, inv=True), ones), 1.0, atol=1e-15)


@pytest.mark.parametrize("prec,tol", [(D, 1e-12), (S, 1e-5)])
def test_fft_round_trip_linearity_parseval(prec, tol):
    """SPEC.md:130-134 / acceptance 9, 100 random batches per precision."""
    rng = np.random.default_rng(3)
    dt = np.float64 if prec == D else np.float32
    for _ in range(100):
        L = 2 * int(rng.integers(1, 300))
        b = int(rng.integers(1, 5))
        x = rng.standard_normal(L * b).astype(dt)
        X = F.forward_real_batched(plan(L, b, prec), x)
        assert rel(F.inverse_real_batched(plan(L, b, prec, inv=True), X), x) <= tol
    L, b = 512, 3
    x, y = rng.standard_normal(L * b), rng.standard_normal(L * b)
    P = plan(L, b)
    assert rel(F.forward_real_batched(P, 1.5 * x - 2 * y),
               1.5 * F.forward_real_batched(P, x) - 2 * F.forward_real_batched(P, y)) < 1e-12
    Xs = F.forward_real_batched(P, x).reshape(b, -1)
    e = (np.abs(Xs[:, 0]) ** 2 + np.abs(Xs[:, -1]) ** 2 + 2 * np.sum(np.abs(Xs[:, 1:-1]) ** 2, axis=1)) / L
    assert np.allclose(e, np.sum(x.reshape(b, -1) ** 2, axis=1), rtol=1e-10)


def test_fft_rejects_bad_plans():
    with pytest.raises(ValueError):
        F.FftPlan(7, 1, D, F.FftDirection.Forward)
    with pytest.raises(ValueError):
        F.forward_real_batched(plan(8, 2), np.zeros(15))


def test_gemv_reference_golden():
    g = golden("gemv")
    for dt in "sdcz":
        for mode in (0, 1, 2):
            A, x, want = g[f"{dt}{mode}_A"], g[f"{dt}{mode}_x"], g[f"{dt}{mode}_y"]
            xl, yl = (13, 7) if mode == 0 else (7, 13)
            for simple in (False, True):
                y, used = F.gemv_batched(F.GemvMode(mode), dt, 7, 13, 3, 7, 91, A, xl, x, yl, force_simple=simple)
                assert used == (1 if simple else 2 if mode else 0)  # 2: small-problem (Conj)Trans kernel
                assert rel(y, want) <= 16 * np.finfo(np.float32 if dt in "sc" else np.float64).eps * 7, (dt, mode)


def _rand(rng, n, dt):
    npdt = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}[dt]
    v = rng.standard_normal(n)
    if dt in "cz":
        v = v + 1j * rng.standard_normal(n)
    return v.astype(npdt)


def test_gemv_shapes_vs_reference_naive(ref):
    """Acceptance 4: within 16*eps*m of the naive kernel over
    random shapes incl. the paper family m=100, n=5000, batch=201."""
    rng = np.random.default_rng(4)
    shapes = [(100, 5000, 201, "c", 2), (100, 5000, 20, "z", 2), (100, 5000, 20, "z", 0), (10, 1000, 100, "c", 2),
              (1, 64, 100, "d", 1), (600, 300, 5, "z", 0), (600, 300, 5, "z", 2), (1000, 70, 3, "s", 0),
              (33, 33, 9, "d", 0), (2, 1, 1, "c", 0), (5, 3, 2, "s", 1)]
    for _ in range(40):
        m, n = int(rng.integers(1, 200)), int(rng.integers(1, 400))
        shapes.append((m, n, int(rng.integers(1, 12)), "sdcz"[int(rng.integers(4))], int(rng.integers(3))))
    for m, n, b, dt, mode in shapes:
        lda = m + int(rng.integers(0, 3))
        sa = lda * n + int(rng.integers(0, 5))
        xl, yl = (n, m) if mode == 0 else (m, n)
        A = _rand(rng, (b - 1) * sa + lda * (n - 1) + m, dt)
        x = _rand(rng, b * xl, dt)
        want = np.zeros(b * yl, dtype=A.dtype)
        ref.gemv(0, mode, dt, m, n, b, lda, sa, A, xl, x, yl, want)
        got, used = F.gemv_batched(F.GemvMode(mode), dt, m, n, b, lda, sa, A, xl, x, yl)
        eps = np.finfo(np.float32 if dt in "sc" else np.float64).eps
        scale = np.abs(A).max() * np.abs(x).max() * m if mode else np.abs(A).max() * np.abs(x).max() * n
        err = np.abs(got - want).max() / max(scale, 1e-30)
        assert err <= 16 * eps * max(m, n), (m, n, b, dt, mode, err)


def test_conjtrans_on_real_equals_trans_bitwise():
    rng = np.random.default_rng(5)
    for dt in "sd":
        A, x = _rand(rng, 37 * 50 * 4, dt), _rand(rng, 37 * 4, dt)
        t, _ = F.gemv_batched(F.GemvMode.Trans, dt, 37, 50, 4, 37, 37 * 50, A, 37, x, 50)
        c, _ = F.gemv_batched(F.GemvMode.ConjTrans, dt, 37, 50, 4, 37, 37 * 50, A, 37, x, 50)
        assert np.array_equal(t, c)


def test_gemv_spec_examples():
    y, _ = F.gemv_batched(F.GemvMode.NoTrans, "d", 3, 3, 2, 3, 9, np.tile(np.eye(3).T.reshape(-1), 2), 3,
                          np.tile([1.0, 2.0, 3.0], 2), 3)
    assert np.array_equal(y, np.tile([1.0, 2.0, 3.0], 2))
    A = np.array([1j, 0, 0, 1j], dtype=np.complex128)
    y, _ = F.gemv_batched(F.GemvMode.ConjTrans, "z", 2, 2, 1, 2, 4, A, 2, np.ones(2, dtype=np.complex128), 2)
    assert np.array_equal(y, np.array([-1j, -1j]))
    with pytest.raises(ValueError):
        F.gemv_batched(F.GemvMode.NoTrans, "d", 3, 3, 1, 2, 9, np.zeros(9), 3, np.zeros(3), 3)


def test_conjtrans_resident_x_matches_per_stage_x(monkeypatch):
    """x_b resident in shared memory (copied once per batch entry) gives the
    same bits as re-copying it with every stage, incl. tall columns (multi-warp
    per column) and pieces that start mid batch."""
    rng = np.random.default_rng(9)
    monkeypatch.setenv("FMV_SBGEMV_SMALL", "0")  # (the staged kernel is the one under test)
    for m, n, b, dt in ((600, 3000, 3, "z"), (1000, 700, 2, "d"), (100, 5000, 4, "c"), (37, 900, 5, "z")):
        A = _rand(rng, m * n * b, dt)
        x = _rand(rng, m * b, dt)
        out = {}
        for flag in ("0", "1"):
            monkeypatch.setenv("FMV_SBGEMV_XRES", flag)
            out[flag], used = F.gemv_batched(F.GemvMode.ConjTrans, dt, m, n, b, m, m * n, A, m, x, n)
            assert used == 0
        assert np.array_equal(out["0"], out["1"]), (m, n, b, dt)


@pytest.mark.parametrize("dt", ["s", "d", "c", "z"])
def test_small_conjtrans_kernel_vs_reference_and_staged(ref, monkeypatch, dt):
    """The latency-oriented small-problem (Conj)Trans kernel (C4's m = 10,
    n = 10^3, batch 100 cells): against the reference's naive GEMV and the
    staged TMA kernel, with vector loads (m a multiple of the 16-byte width),
    scalar loads (odd m, padded lda) and the real Trans path."""
    rng = np.random.default_rng(12)
    eps = np.finfo(np.float32 if dt in "sc" else np.float64).eps
    for m, n, b, lda, mode in ((10, 1000, 100, 10, 2), (8, 333, 7, 8, 2), (13, 500, 9, 15, 2), (10, 1000, 100, 10, 1),
                               (64, 129, 3, 64, 2)):
        sa = lda * n
        A = _rand(rng, b * sa, dt)
        x = _rand(rng, b * m, dt)
        want = np.zeros(b * n, dtype=A.dtype)
        ref.gemv(0, mode, dt, m, n, b, lda, sa, A, m, x, n, want)
        got, used = F.gemv_batched(F.GemvMode(mode), dt, m, n, b, lda, sa, A, m, x, n)
        assert used == 2
        scale = np.abs(A).max() * np.abs(x).max() * m
        assert np.abs(got - want).max() / scale <= 16 * eps * m, (m, n, b, dt, mode)
        monkeypatch.setenv("FMV_SBGEMV_SMALL", "0")
        staged, used0 = F.gemv_batched(F.GemvMode(mode), dt, m, n, b, lda, sa, A, m, x, n)
        monkeypatch.delenv("FMV_SBGEMV_SMALL")
        assert used0 == 0
        assert np.abs(got - staged).max() / scale <= 16 * eps * m
