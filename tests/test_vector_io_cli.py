"""FMV1 vector persistence and the fft_matvec CLI (SPEC.md cli module,
SURVEY.md §8 f4). CPU: acceptance 12 (100 random vectors over every
layout/precision/domain code round-trip bitwise), the named decode errors,
byte-for-byte agreement of the Python and C++ writers, CLI usage errors.
GPU: the CLI's -raw CSV schema, -s output files against the library's own
matvec results, -sweep CSV read back by parse_sweep_csv, -p partitions."""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import ROOT

CLI = os.path.join(ROOT, "build", "fft_matvec")
CPP = os.path.join(ROOT, "build", "fftmv_cpp_tests")


def test_fmv1_round_trip_acceptance12(tmp_path):
    rng = np.random.default_rng(12)
    for i in range(100):
        lay, prec, dom = (F.Layout.SOTI, F.Layout.TOSI)[i % 2], (F.Precision.Double, F.Precision.Single)[(i // 2) % 2], \
            (F.Domain.Time, F.Domain.Frequency)[(i // 4) % 2]
        s, t = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        n = s * t * (2 if dom == F.Domain.Frequency else 1)
        data = rng.standard_normal(n).astype(np.float64 if prec == F.Precision.Double else np.float32)
        v = F.BlockVector(s, t, lay, prec, dom, data)
        p = str(tmp_path / f"v{i}.fmv")
        F.save_vector(p, v)
        w = F.load_vector(p)
        assert (w.space_extent, w.time_extent, w.layout, w.precision, w.domain) == (s, t, lay, prec, dom)
        assert w.data.dtype == data.dtype and w.data.tobytes() == data.tobytes()
        assert os.path.getsize(p) == 44 + data.nbytes


def test_fmv1_errors():
    good = F.encode_vector(F.BlockVector.time_double(2, 3, np.arange(6.0)))
    with pytest.raises(ValueError, match="bad magic"):
        F.decode_vector(b"")
    with pytest.raises(ValueError, match="bad magic"):
        F.decode_vector(b"FMV2" + good[4:])
    with pytest.raises(ValueError, match="truncated file"):
        F.decode_vector(good[:20])
    with pytest.raises(ValueError, match="truncated/oversized"):
        F.decode_vector(good[:-8])
    hdr_f32 = bytearray(good)
    hdr_f32[4 + 24] = 1  # header says f32 but payload sized for f64 (SPEC.md example)
    with pytest.raises(ValueError, match="truncated/oversized"):
        F.decode_vector(bytes(hdr_f32))
    bad = bytearray(good)
    bad[4 + 32] = 7
    with pytest.raises(ValueError, match="domain code out of range"):
        F.decode_vector(bytes(bad))


def test_fmv1_python_and_cpp_writers_agree(tmp_path):
    if not os.path.exists(CPP):
        pytest.skip("build/fftmv_cpp_tests not built (make cpp)")
    p = str(tmp_path / "cpp.fmv")
    r = subprocess.run([CPP], env={**os.environ, "FMV1_OUT": p}, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    want = F.encode_vector(F.BlockVector.time_double(4, 9, F.uniform_fill(36, 2025)))
    assert open(p, "rb").read() == want


def test_cli_usage_errors():
    if not os.path.exists(CLI):
        pytest.skip("build/fft_matvec not built (make cli)")
    for args, msg in ((["-prec", "xyzzy"], "position 1"), (["-nm", "0"], "-nm"), (["-bogus"], "unknown flag"),
                      (["-tol"], "missing"), (["-nm", "4", "-p", "5"], "more workers")):
        r = subprocess.run([CLI] + args, capture_output=True, text=True)
        assert r.returncode == 2 and msg in r.stderr, (args, r.stderr)


@pytest.mark.gpu
def test_cli_raw_save_sweep_partition(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("build/fft_matvec not built (make cli)")
    nm, nd, nt = 50, 5, 16
    args = [CLI, "-nm", str(nm), "-nd", str(nd), "-Nt", str(nt), "-reps", "3", "-warmup", "1"]
    r = subprocess.run(args + ["-prec", "ddddd", "-raw", "-s", str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert list(rows[0].keys()) == ["matvec", "phase", "mean_s", "min_s", "max_s"]
    assert [x["matvec"] for x in rows] == ["forward"] * 6 + ["adjoint"] * 6
    assert rows[5]["phase"] == "total" and all(float(x["min_s"]) <= float(x["mean_s"]) <= float(x["max_s"]) for x in rows)
    # saved outputs equal the library's own matvecs on the same seeded inputs, bitwise
    S = 20250814
    col = F.uniform_fill(nm * nd * nt, F.seed_stream(S, 0))
    op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
    fo, ao = F.load_vector(str(tmp_path / "forward_output.fmv")), F.load_vector(str(tmp_path / "adjoint_output.fmv"))
    assert np.array_equal(fo.data, F.forward_matvec(op, F.uniform_fill(nm * nt, F.seed_stream(S, 1))).output.data)
    assert np.array_equal(ao.data, F.adjoint_matvec(op, F.uniform_fill(nd * nt, F.seed_stream(S, 2))).output.data)
    r = subprocess.run(args + ["-sweep", "-rand", "-raw", "-tol", "1e-5"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    sections = []
    for line in r.stdout.splitlines():
        if line.startswith("#"):
            sections.append([line])
        else:
            sections[-1].append(line)
    assert [sec[0].split()[1] for sec in sections] == ["forward", "adjoint"]
    for sec in sections:
        back = F.parse_sweep_csv("\n".join(sec))
        assert len(back) == 32 and back[0].config.render() == "ddddd" and back[0].rel_error == 0.0
        chosen = sec[0].split("chosen=")[1].split()[0]
        assert next(b for b in back if b.config.render() == chosen).rel_error <= 1e-5
    r = subprocess.run(args + ["-p", "4", "-prec", "dddds", "-s", str(tmp_path / "p4")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    pf = F.load_vector(str(tmp_path / "p4" / "forward_output.fmv")).data
    assert 0 < np.linalg.norm(pf - fo.data) / np.linalg.norm(fo.data) <= 1e-4
