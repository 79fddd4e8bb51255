"""C3 (BASELINE.json configs[2]) at full size: the mixed-precision sweep at the
C2 shape (Nm=5000, Nd=100, Nt=1000) with the sweep's own fill
(non_representable_fill, sweep.hpp:32-46), all 32 reference configs for F and
F*, against the LIVE reference (oracle/_ref) on the same inputs.

Tolerance (SURVEY.md §8 d): every GPU output's relative L2 error against the
CPU reference's 'ddddd' output must be <= max(2 * err_ref(cfg), 1e-12), where
err_ref(cfg) is the reference's own error for that config against its
'ddddd'. The fp16 'h' extension has no reference counterpart: its stated
bound is 5e-3. The GPU runs through the host-I/O entry point (fmv_matvec,
overlapped column chunks), the reference configs run concurrently on the
host cores."""
import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import SEED, configs32, rel

pytestmark = pytest.mark.gpu

NM, ND, NT = 5000, 100, 1000
HALF_TOL = 5e-3


@pytest.fixture(scope="module")
def c3():
    from oracle.oracle import have_ref, ref

    if not have_ref():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    R = ref()
    col = R.non_representable_fill(NM * ND * NT, R.seed_stream(SEED, 0))
    m = R.non_representable_fill(NM * NT, R.seed_stream(SEED, 1))
    d = R.non_representable_fill(ND * NT, R.seed_stream(SEED, 2))
    rop = R.setup_operator(NM, ND, NT, col)
    jobs = [(k, c, m if k == 0 else d) for c in configs32() for k in (0, 1)]
    outs = R.matvec_many(rop, jobs)
    ref_out = {(k, c): o for (k, c, _), o in zip(jobs, outs)}
    del rop
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), col))
    return op, m, d, ref_out


def test_c3_all_32_configs_vs_live_reference(c3):
    op, m, d, ref_out = c3
    base = {0: ref_out[(0, "ddddd")], 1: ref_out[(1, "ddddd")]}
    rows = []
    for cfg in configs32():
        for kind, x, fn in ((0, m, F.forward_matvec), (1, d, F.adjoint_matvec)):
            got = fn(op, x, cfg, timings=False).output.data
            err = rel(got, base[kind])
            err_ref = rel(ref_out[(kind, cfg)], base[kind])
            rows.append((cfg, kind, err, err_ref))
    bad = [r for r in rows if not r[2] <= max(2 * r[3], 1e-12)]
    assert not bad, bad
    # the fp32 SBGEMV configs land below the reference's sequential fp32 sums
    # (DESIGN.md §3.1): F ddsdd ~1e-7 vs the reference's 1.27e-6
    e = {(c, k): (er, eref) for c, k, er, eref in rows}
    assert e[("ddsdd", 0)][0] < 0.5 * e[("ddsdd", 0)][1]


def test_c3_half_extension(c3):
    op, m, d, ref_out = c3
    base = {0: ref_out[(0, "ddddd")], 1: ref_out[(1, "ddddd")]}
    for cfg in ("ddhdd", "hdhdd", "ddhdh", "hdhdh", "sshsd", "dshsd"):
        ef = rel(F.forward_matvec(op, m, cfg, timings=False).output.data, base[0])
        ea = rel(F.adjoint_matvec(op, d, cfg, timings=False).output.data, base[1])
        assert 0 < ef <= HALF_TOL and 0 < ea <= HALF_TOL, (cfg, ef, ea)


def test_c3_fp64_accumulate_variant(c3):
    """The 'm' SBGEMV variant (fp32 operator and spectrum, fp64 accumulation;
    SURVEY.md App. A4): at C2 its error is the input-rounding floor, below the
    fp32-accumulating 's' config and below tau = 1e-7, for F and F*."""
    op, m, d, ref_out = c3
    base = {0: ref_out[(0, "ddddd")], 1: ref_out[(1, "ddddd")]}
    for kind, x, fn in ((0, m, F.forward_matvec), (1, d, F.adjoint_matvec)):
        em = rel(fn(op, x, "ddmdd", timings=False).output.data, base[kind])
        es = rel(fn(op, x, "ddsdd", timings=False).output.data, base[kind])
        assert 0 < em < 1e-7 and em < es, (kind, em, es)
        for cfg in ("dsmdd", "ssmss", "ddmds"):
            e = rel(fn(op, x, cfg, timings=False).output.data, base[kind])
            assert e <= 2 * rel(ref_out[(kind, cfg.replace("m", "s"))], base[kind]), (kind, cfg, e)
