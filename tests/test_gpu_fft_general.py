"""General-length FFTs (fft.hpp:32-95 plans every even L): the runtime-plan
register kernels (k_r2c_rt / k_c2r_rt), the legacy two-buffer shared-memory
kernels and the HBM-scratch Stockham path, against the reference's own FFT
(oracle/_ref, FFTW API over MKL) and against each other, and whole matvecs at
n_t outside the two specialised lengths (1000, 100) against the reference.
Run with -m gpu."""
import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import make_inputs, rel

pytestmark = pytest.mark.gpu

D, S = F.Precision.Double, F.Precision.Single
# complex lengths N = L/2: radix-16 / 10 / 8 / 5 / 7 / 3 / 2 register plans, a
# length whose plan needs > 512 threads (10^4), a prime inside the legacy
# capacity (1009) and one beyond it in fp64 (8209)
NS = [2, 3, 5, 7, 8, 12, 16, 24, 49, 64, 100, 125, 250, 256, 343, 500, 512, 768, 1000, 1024, 2000, 2048, 3000,
      4096, 5000, 8192, 1009, 10000, 8209]


def plan(L, b, p=D, inv=False):
    return F.FftPlan(L, b, p, F.FftDirection.Inverse if inv else F.FftDirection.Forward)


@pytest.mark.parametrize("prec", [D, S])
def test_fft_lengths_vs_reference(ref, prec):
    rng = np.random.default_rng(7)
    tol_f, tol_i = (1e-12, 1e-12) if prec == D else (2e-5, 2e-5)
    dt = np.float64 if prec == D else np.float32
    for N in NS:
        L, b = 2 * N, 3
        x = rng.uniform(-1, 1, L * b).astype(dt)
        want = ref.fft_forward(L, b, x, 1 if prec == D else 0)
        got = F.forward_real_batched(plan(L, b, prec), x)
        assert rel(got, want) <= tol_f, (N, rel(got, want))
        back = F.inverse_real_batched(plan(L, b, prec, inv=True), got)
        assert rel(back, x) <= tol_i, (N, rel(back, x))


@pytest.mark.parametrize("N", [8, 100, 343, 1000, 1024, 3000, 4096, 8192])
def test_fft_paths_agree(monkeypatch, N):
    """The same transforms through every kernel family that can run them."""
    rng = np.random.default_rng(N)
    L, b = 2 * N, 5
    x = rng.standard_normal(L * b)
    outs = {}
    for path in ("auto", "rt", "legacy", "global"):
        monkeypatch.setenv("FMV_FFT_PATH", path)
        outs[path] = (F.forward_real_batched(plan(L, b), x), F.inverse_real_batched(plan(L, b, inv=True),
                                                                                    np.fft.rfft(x.reshape(b, L)).reshape(-1)))
    monkeypatch.delenv("FMV_FFT_PATH")
    base_f, base_i = outs["global"]
    assert rel(base_f, np.fft.rfft(x.reshape(b, L)).reshape(-1)) <= 1e-12
    for path, (f, i) in outs.items():
        assert rel(f, base_f) <= 1e-13, (N, path)
        assert rel(i, base_i) <= 1e-13, (N, path)


@pytest.mark.parametrize("nt", [512, 1024, 2000, 4096, 8192, 343, 3000, 1009, 8209])
def test_matvec_general_nt_vs_reference(ref, nt):
    """Whole F / F* matvecs (fused pad / cast / reorder / unpad in the general
    kernels, operator setup through the time-outer path) at n_t outside the
    specialised 1000 / 100 against the reference itself."""
    nm, nd = 6, 3
    col, m, d = make_inputs(F, nm, nd, nt, "nonrep")
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    rop = ref.setup_operator(nm, nd, nt, col)
    assert rel(op.bins_double, rop.bins()) <= 1e-13
    rf, ra = ref.matvec(rop, 0, "ddddd", m), ref.matvec(rop, 1, "ddddd", d)
    assert rel(F.forward_matvec(op, m).output.data, rf) <= 1e-12
    assert rel(F.adjoint_matvec(op, d).output.data, ra) <= 1e-12
    for cfg in ("dsddd", "ddsdd", "dddsd", "sssss", "sdddd", "dddds"):
        ef = max(2 * rel(ref.matvec(rop, 0, cfg, m), rf), 1e-12)
        ea = max(2 * rel(ref.matvec(rop, 1, cfg, d), ra), 1e-12)
        assert rel(F.forward_matvec(op, m, cfg).output.data, rf) <= ef, (nt, cfg)
        assert rel(F.adjoint_matvec(op, d, cfg).output.data, ra) <= ea, (nt, cfg)
    assert rel(F.forward_matvec(op, m, "hdhdh").output.data, rf) <= 5e-3
