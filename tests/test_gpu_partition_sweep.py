"""GPU: the 1 x p partition (in-process and through the NCCL entry point at
world size 1), the mixed-precision sweep / Pareto front, the C++ drop-in
binary and the graft smoke entry. Run with -m gpu."""
import os
import subprocess

import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import ROOT, golden, make_inputs, rel

pytestmark = pytest.mark.gpu


def test_partitioned_vs_reference_golden():
    """Acceptance 8: p in {1,2,4,8,16} at 64/4/32."""
    g = golden("partition")
    nm, nd, nt = 64, 4, 32
    col, m, d = make_inputs(F, nm, nd, nt)
    dims = F.ProblemDims(nm, nd, nt)
    serial = F.setup_operator(F.BlockColumn(dims, col))
    sf, sa = F.forward_matvec(serial, m).output.data, F.adjoint_matvec(serial, d).output.data
    for p in (1, 2, 4, 8, 16):
        pop = F.setup_partitioned(F.BlockColumn(dims, col), F.Grid1xP.split(p, nm))
        for cfg in ("ddddd", "dddds", "sdddd"):
            pf = F.forward_matvec_partitioned(pop, m, cfg).output.data
            pa = F.adjoint_matvec_partitioned(pop, d, cfg).output.data
            if cfg == "ddddd":
                assert rel(pf, g[f"p{p}_F_ddddd"]) <= 1e-12 and rel(pa, g[f"p{p}_A_ddddd"]) <= 1e-12
                assert rel(pf, sf) <= 1e-12 and rel(pa, sa) <= 1e-12
                if p == 1:
                    assert np.array_equal(pf, sf) and np.array_equal(pa, sa)
            elif cfg == "dddds":
                assert 0 < rel(pf, sf) <= 1e-4
            else:  # sdddd: the broadcast cast happens once, worker-count independent
                assert rel(pa, g[f"p{p}_A_sdddd"]) <= 1e-12


def test_native_partition_entry_world1_is_bitwise_serial():
    nm, nd, nt = 40, 6, 30
    col, m, d = make_inputs(F, nm, nd, nt)
    dims = F.ProblemDims(nm, nd, nt)
    op = F.setup_operator(F.BlockColumn(dims, col))
    dm = F.DistributedMatvec(dims, 0, 1, shard=op, transport="native")
    for cfg in ("ddddd", "dssds", "sdddd", "hdhdh"):
        assert np.array_equal(dm.forward(m, cfg), F.forward_matvec(op, m, cfg).output.data), cfg
        want = F.adjoint_matvec(op, F.round_to(d, cfg[0]), "d" + cfg[1:]).output.data
        assert np.array_equal(dm.adjoint(d, cfg), want), cfg
    dm.close()


def test_grid2d_in_process_vs_serial_and_1xp():
    """pr x pc grid simulated on one GPU. ddddd within 1e-12
    of the serial matvec for every grid; pr = 1 is the 1 x p partition
    bitwise; mixed configs within the serial config's error scale."""
    nm, nd, nt = 60, 9, 100
    col, m, d = make_inputs(F, nm, nd, nt)
    dims = F.ProblemDims(nm, nd, nt)
    serial = F.setup_operator(F.BlockColumn(dims, col))
    sf, sa = F.forward_matvec(serial, m).output.data, F.adjoint_matvec(serial, d).output.data
    for pr, pc in ((1, 1), (1, 3), (2, 1), (2, 2), (3, 4)):
        pop = F.setup_partitioned_2d(F.BlockColumn(dims, col), F.GridPxQ.split(pr, pc, nd, nm))
        for cfg in ("ddddd", "dssdd", "sddds"):
            pf = F.forward_matvec_partitioned_2d(pop, m, cfg).output.data
            pa = F.adjoint_matvec_partitioned_2d(pop, d, cfg).output.data
            if cfg == "ddddd":
                assert rel(pf, sf) <= 1e-12 and rel(pa, sa) <= 1e-12, (pr, pc)
            else:
                ef = rel(F.forward_matvec(serial, m, cfg).output.data, sf)
                ea = rel(F.adjoint_matvec(serial, d, cfg).output.data, sa)
                assert rel(pf, sf) <= 4 * ef + 1e-12 and rel(pa, sa) <= 4 * ea + 1e-12, (pr, pc, cfg)
            if pr == 1:
                q = F.setup_partitioned(F.BlockColumn(dims, col), F.Grid1xP.split(pc, nm))
                assert np.array_equal(pf, F.forward_matvec_partitioned(q, m, cfg).output.data), (pc, cfg)
                assert np.array_equal(pa, F.adjoint_matvec_partitioned(q, d, cfg).output.data), (pc, cfg)


def test_native_grid2d_entry_world1_is_bitwise_serial():
    nm, nd, nt = 40, 6, 30
    col, m, d = make_inputs(F, nm, nd, nt)
    dims = F.ProblemDims(nm, nd, nt)
    op = F.setup_operator(F.BlockColumn(dims, col))
    dm = F.DistributedMatvec2D(dims, 1, 1, 0, shard=op, transport="native")
    for cfg in ("ddddd", "dssds", "sdddd", "hdhdh"):
        assert np.array_equal(dm.forward(m, cfg), F.forward_matvec(op, m, cfg).output.data), cfg
        want = F.adjoint_matvec(op, F.round_to(d, cfg[0]), "d" + cfg[1:]).output.data
        assert np.array_equal(dm.adjoint(d, cfg), want), cfg
    dm.close()


def test_sweep_acceptance5_and_pareto():
    """SPEC.md:544 at 500/20/200, non-representable fill, 32 rows."""
    nm, nd, nt = 500, 20, 200
    col, m, _ = make_inputs(F, nm, nd, nt, "nonrep")
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    rows = F.sweep_operator(op, m, F.MatvecKind.Forward, repetitions=5, warmup=1)
    assert [r.config.render() for r in rows] == [c.render() for c in F.enumerate_configs()]
    assert rows[0].rel_error == 0.0
    assert all(r.rel_error > 0 for r in rows[1:])
    assert next(r for r in rows if r.config.render() == "dssdd").rel_error <= 1e-5
    tol = 1e-5
    best = min((r for r in rows if r.rel_error <= tol), key=lambda r: (r.mean_s, r.rel_error, r.config.render()))
    assert F.optimal_config(rows, tol) == best.config
    front = F.pareto_front(rows)
    assert any(r.config == best.config for r in front)
    rep = F.make_report(F.ProblemDims(nm, nd, nt), F.MatvecKind.Forward, 5, tol, rows)
    assert [r.config for r in F.parse_sweep_csv(F.to_csv(rep))] == [r.config for r in rows]


def test_cpp_dropin_binary_on_gpu():
    exe = os.path.join(ROOT, "build", "fftmv_cpp_tests")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpp"], check=True)
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_graft_smoke():
    import __graft_entry__

    __graft_entry__.smoke()
