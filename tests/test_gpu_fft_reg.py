"""GPU parity of the register-resident radix-10 FFT kernels (k_r2c_reg /
k_c2r_reg, n_t = 1000 and 100) that carry the matvec hot path: against the
reference itself (oracle/_ref) on every precision config, and against the
general mixed-radix kernels (FMV_FFT_LEGACY=1) on the same inputs. Ragged
series counts (Nm, Nd not multiples of the series-per-CTA) exercise the
partial last CTA. Run with -m gpu."""
import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import configs32, make_inputs, rel

pytestmark = pytest.mark.gpu


def _run(op, m, d, cfg):
    return F.forward_matvec(op, m, cfg).output.data, F.adjoint_matvec(op, d, cfg).output.data


@pytest.mark.parametrize("nm,nd,nt", [(37, 5, 1000), (33, 3, 100), (1, 1, 1000)])
def test_reg_fft_all_configs_vs_reference(ref, nm, nd, nt):
    col, m, d = make_inputs(F, nm, nd, nt, "nonrep")
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    rop = ref.setup_operator(nm, nd, nt, col)
    rf, ra = ref.matvec(rop, 0, "ddddd", m), ref.matvec(rop, 1, "ddddd", d)
    for cfg in configs32():
        gf, ga = _run(op, m, d, cfg)
        if cfg == "ddddd":
            assert rel(gf, rf) <= 1e-12 and rel(ga, ra) <= 1e-12
        else:
            ef = max(2 * rel(ref.matvec(rop, 0, cfg, m), rf), 1e-12)
            ea = max(2 * rel(ref.matvec(rop, 1, cfg, d), ra), 1e-12)
            assert rel(gf, rf) <= ef, (cfg, rel(gf, rf), ef)
            assert rel(ga, ra) <= ea, (cfg, rel(ga, ra), ea)


@pytest.mark.parametrize("nt", [1000, 100])
def test_reg_fft_matches_legacy_kernels(monkeypatch, nt):
    nm, nd = 45, 7
    col, m, d = make_inputs(F, nm, nd, nt)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    for cfg in ("ddddd", "dsddd", "dddsd", "sssss", "hdhdh"):
        monkeypatch.setenv("FMV_FFT_LEGACY", "0")
        gf, ga = _run(op, m, d, cfg)
        monkeypatch.setenv("FMV_FFT_LEGACY", "1")
        lf, la = _run(op, m, d, cfg)
        tol = 1e-14 if cfg == "ddddd" else 2e-6 if "h" not in cfg else 2e-3
        assert rel(gf, lf) <= tol and rel(ga, la) <= tol, cfg
    monkeypatch.setenv("FMV_FFT_LEGACY", "0")
    assert np.array_equal(_run(op, m, d, "ddddd")[0], _run(op, m, d, "ddddd")[0])  # deterministic
