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


@pytest.mark.parametrize("nm", [1030, 1024])
def test_big_fft_kernels_all_configs_vs_reference(ref, nm):
    """The big transforms (>= 1024 series at n_t = 1000: F's r2c over Nm
    series, F*'s c2r over Nm series) have three kernel sets (FMV_FFT_BIG):
    the persistent prefetching ones (default, fmv_fft_stream.cuh), the
    paired-butterfly ones (fmv_fft_pair.cuh) and the one-shot k_*_reg.
    Nm = 1030 leaves a partial last tile for every series-per-tile choice.
    Every config of each set against the reference itself; the sets against
    each other on the same inputs; determinism."""
    import os

    nd, nt = 3, 1000
    col, m, d = make_inputs(F, nm, nd, nt, "nonrep")
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    rop = ref.setup_operator(nm, nd, nt, col)
    jobs = [(k, c, m if k == 0 else d) for c in configs32() for k in (0, 1)]
    want = {(k, c): o for (k, c, _), o in zip(jobs, ref.matvec_many(rop, jobs))}
    rf, ra = want[(0, "ddddd")], want[(1, "ddddd")]
    got = {}
    try:
        for kind in ("stream", "pair", "reg"):
            os.environ["FMV_FFT_BIG"] = kind
            for cfg in configs32():
                gf, ga = _run(op, m, d, cfg)
                ef = max(2 * rel(want[(0, cfg)], rf), 1e-12)
                ea = max(2 * rel(want[(1, cfg)], ra), 1e-12)
                assert rel(gf, rf) <= ef, (kind, cfg, rel(gf, rf), ef)
                assert rel(ga, ra) <= ea, (kind, cfg, rel(ga, ra), ea)
            for cfg in ("ddddd", "dssdd", "sssss", "ddhdd", "hdhdh"):
                got[(kind, cfg)] = _run(op, m, d, cfg)
            assert np.array_equal(_run(op, m, d, "ddddd")[1], got[(kind, "ddddd")][1])  # deterministic
    finally:
        del os.environ["FMV_FFT_BIG"]
    for kind in ("stream", "pair"):
        for cfg in ("ddddd", "dssdd", "sssss", "ddhdd", "hdhdh"):
            (pf, pa), (qf, qa) = got[(kind, cfg)], got[("reg", cfg)]
            tol = 1e-14 if cfg == "ddddd" else 2e-6 if "h" not in cfg else 2e-3
            assert rel(pf, qf) <= tol and rel(pa, qa) <= tol, (kind, cfg, rel(pf, qf), rel(pa, qa))
