"""GPU parity at BASELINE.json configs[1] (C2: Nm=5000, Nd=100, Nt=1000),
against the reference binary when built (else size-independent properties
only). Run with -m gpu."""
import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import make_inputs, rel

pytestmark = pytest.mark.gpu

NM, ND, NT = 5000, 100, 1000


@pytest.fixture(scope="module")
def c2():
    col, m, d = make_inputs(F, NM, ND, NT)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(NM, ND, NT), col))
    return col, m, d, op


def test_c2_properties(c2):
    col, m, d, op = c2
    f = F.forward_matvec(op, m).output.data
    a = F.adjoint_matvec(op, d).output.data
    assert abs(f @ d - m @ a) <= 1e-11 * abs(f @ d)  # adjointness at full size
    assert np.array_equal(f, F.forward_matvec(op, m).output.data)  # bitwise determinism
    assert np.array_equal(a, F.adjoint_matvec(op, d).output.data)
    m2 = F.uniform_fill(NM * NT, 5)
    assert rel(F.forward_matvec(op, m + m2).output.data, f + F.forward_matvec(op, m2).output.data) <= 1e-12


def test_c2_vs_reference(c2):
    from oracle.oracle import have_ref, ref

    if not have_ref():
        pytest.skip("oracle/_ref not built")
    col, m, d, op = c2
    R = ref()
    rop = R.setup_operator(NM, ND, NT, col)
    assert rel(op.bins_double, rop.bins()) <= 1e-13
    rf, ra = R.matvec(rop, 0, "ddddd", m), R.matvec(rop, 1, "ddddd", d)
    assert rel(F.forward_matvec(op, m).output.data, rf) <= 1e-12
    assert rel(F.adjoint_matvec(op, d).output.data, ra) <= 1e-12
    # mixed precision: within max(2 * err_ref, 1e-12) of the reference ddddd output
    for cfg in ("dssdd", "ddssd", "dddds"):
        ef = rel(F.forward_matvec(op, m, cfg).output.data, rf)
        ea = rel(F.adjoint_matvec(op, d, cfg).output.data, ra)
        assert ef <= max(2 * rel(R.matvec(rop, 0, cfg, m), rf), 1e-12), cfg
        assert ea <= max(2 * rel(R.matvec(rop, 1, cfg, d), ra), 1e-12), cfg
    for cfg in ("ddhdd", "hdhdh"):
        assert rel(F.forward_matvec(op, m, cfg).output.data, rf) <= 5e-3
        assert rel(F.adjoint_matvec(op, d, cfg).output.data, ra) <= 5e-3


def test_c5_shard_properties():
    """BASELINE.json configs[4] per-GPU shard (Nm=5000, Nd=600, Nt=1000; 48 GB fp64
    operator): the reference cannot hold it on the host, so check size-independent
    properties at full size -- adjointness, linearity, bitwise determinism -- and
    that the block path agrees with the single-RHS path."""
    import psutil

    nm, nd, nt = 5000, 600, 1000
    if psutil.virtual_memory().available < 64 * 2 ** 30:
        pytest.skip("needs ~30 GB of free host memory for the synthetic block column")
    col, m, d = make_inputs(F, nm, nd, nt)
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    del col
    f = F.forward_matvec(op, m).output.data
    a = F.adjoint_matvec(op, d).output.data
    assert abs(f @ d - m @ a) <= 1e-11 * abs(f @ d)
    assert np.array_equal(f, F.forward_matvec(op, m).output.data)
    assert np.array_equal(a, F.adjoint_matvec(op, d).output.data)
    m2 = F.uniform_fill(nm * nt, 7)
    assert rel(F.forward_matvec(op, m + m2).output.data, f + F.forward_matvec(op, m2).output.data) <= 1e-12
    D = np.stack([d, -2 * d])
    B = F.adjoint_matvec_block(op, D)
    assert rel(B[0], a) <= 1e-14 and rel(B[1], -2 * a) <= 1e-14
