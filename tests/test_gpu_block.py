"""GPU checks of the block (multi-RHS) matvec: each RHS of
fmv_matvec_block against the single-RHS path on the same inputs and against
the reference itself (oracle/_ref) for a few RHS; K = 1..19 (1 launch with
KR = 2/4/8, and several launches past 8 RHS); ragged Nm, Nd and column
counts; device and host I/O; fp16 SBGEMV configs (routed through the
single-RHS path). Run with -m gpu."""
import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import make_inputs, rel

pytestmark = pytest.mark.gpu

# summation-order tolerance of a block RHS vs the single-RHS kernel, by SBGEMV precision
TOL = {"d": 1e-14, "s": 2e-6, "h": 0.0}


def _op(nm, nd, nt, fill="uni"):
    col, _, _ = make_inputs(F, nm, nd, nt, fill)
    return F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col)), col


def _rhs(K, n, seed):
    return np.stack([F.uniform_fill(n, F.seed_stream(seed, 10 + r)) for r in range(K)])


@pytest.mark.parametrize("nm,nd,nt", [(37, 5, 100), (300, 20, 64), (45, 7, 1000), (40, 150, 32)])
@pytest.mark.parametrize("K", [2, 3, 8, 11])
def test_block_matches_single_rhs(nm, nd, nt, K):
    op, _ = _op(nm, nd, nt)
    M, D = _rhs(K, nm * nt, 1), _rhs(K, nd * nt, 2)
    for cfg in ("ddddd", "dssdd", "sssss", "ddsdd"):
        tol = TOL[cfg[2]] if cfg[2] == "d" else max(TOL[cfg[2]], 1e-12)
        BF, BA = F.forward_matvec_block(op, M, cfg), F.adjoint_matvec_block(op, D, cfg)
        assert BF.shape == (K, nd * nt) and BA.shape == (K, nm * nt)
        for r in range(K):
            sf = F.forward_matvec(op, M[r], cfg).output.data
            sa = F.adjoint_matvec(op, D[r], cfg).output.data
            assert rel(BF[r], sf) <= tol, (cfg, r, rel(BF[r], sf))
            assert rel(BA[r], sa) <= tol, (cfg, r, rel(BA[r], sa))
        assert np.array_equal(F.forward_matvec_block(op, M, cfg), BF)  # deterministic
        assert np.array_equal(F.adjoint_matvec_block(op, D, cfg), BA)


def test_block_vs_reference(ref):
    nm, nd, nt = 64, 6, 1000
    op, col = _op(nm, nd, nt, "nonrep")
    rop = ref.setup_operator(nm, nd, nt, col)
    M, D = _rhs(5, nm * nt, 3), _rhs(5, nd * nt, 4)
    BF, BA = F.forward_matvec_block(op, M), F.adjoint_matvec_block(op, D)
    for r in range(5):
        assert rel(BF[r], ref.matvec(rop, 0, "ddddd", M[r])) <= 1e-12
        assert rel(BA[r], ref.matvec(rop, 1, "ddddd", D[r])) <= 1e-12
    for cfg in ("dssdd", "ddssd"):
        BF, BA = F.forward_matvec_block(op, M, cfg), F.adjoint_matvec_block(op, D, cfg)
        for r in (0, 4):
            rf, ra = ref.matvec(rop, 0, "ddddd", M[r]), ref.matvec(rop, 1, "ddddd", D[r])
            assert rel(BF[r], rf) <= max(2 * rel(ref.matvec(rop, 0, cfg, M[r]), rf), 1e-12), cfg
            assert rel(BA[r], ra) <= max(2 * rel(ref.matvec(rop, 1, cfg, D[r]), ra), 1e-12), cfg


def test_block_device_io_half_and_edge_cases():
    import torch

    nm, nd, nt = 50, 4, 100
    op, _ = _op(nm, nd, nt)
    M, D = _rhs(4, nm * nt, 5), _rhs(4, nd * nt, 6)
    hf = F.forward_matvec_block(op, M)
    df = F.forward_matvec_block(op, torch.from_numpy(M).cuda())
    assert np.array_equal(df.cpu().numpy(), hf)
    for cfg in ("ddhdd", "hdhdh"):  # fp16 SBGEMV: K single-RHS pipelines, bitwise equal to them
        B = F.adjoint_matvec_block(op, D, cfg)
        for r in range(4):
            assert np.array_equal(B[r], F.adjoint_matvec(op, D[r], cfg).output.data)
    assert F.forward_matvec_block(op, M[:0]).shape == (0, nd * nt)
    B1 = F.forward_matvec_block(op, M[:1])
    assert rel(B1[0], F.forward_matvec(op, M[0]).output.data) == 0.0  # K = 1 is the single-RHS path
    with pytest.raises(ValueError):
        F.forward_matvec_block(op, M[:, :-1])
    with pytest.raises(ValueError):
        F.forward_matvec_block(op, M, "ddxdd")
