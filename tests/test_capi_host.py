"""C ABI and host-side API checks that need no GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2508_10202_b200 as F
from conftest import ROOT, SEED, golden, rel


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fftmv_cuda.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)  # declarations only, not prose
    return sorted(set(re.findall(r"\b(fmv_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = F.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", F.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(fmv_\w+)", out))
    declared = header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(lib, s)
    assert set(F._capi.exported_symbols()) <= set(declared)


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(F.FmvError):
        F.Context(0)


def test_fills_bitwise_vs_reference_golden():
    g = golden("fills")
    assert np.array_equal(F.uniform_fill(64, 7), g["fill_uniform_seed7"])
    assert np.array_equal(F.uniform_fill(64, 7, 0.0, 5.0), g["fill_uniform_seed7_0_5"])
    assert np.array_equal(F.non_representable_fill(64, 9), g["fill_nonrep_seed9"])
    assert [F.seed_stream(SEED, k) for k in range(4)] == [int(v) for v in g["seed_stream"]]
    with pytest.raises(ValueError):
        F.non_representable_fill(0, 1)


def test_relative_error():
    x = np.array([1.0, 2.0, 3.0])
    assert F.relative_error(x, x) == 0.0
    assert F.relative_error(2 * x, x) == pytest.approx(1.0)
    e = np.array([1.0, 0.0, 0.0])
    assert F.relative_error(e + np.array([1e-9, 0, 0]), e) == pytest.approx(1e-9, rel=1e-6)
    with pytest.raises(ValueError):
        F.relative_error(x, np.zeros(3))
    with pytest.raises(ValueError):
        F.relative_error(x, x[:2])


def test_host_copy():
    """fmv_host_copy: the library's host-pool memcpy (fills the drop-in's result
    vectors from its pinned buffer); sizes below and above the split threshold,
    unaligned offsets, and the null-pointer error."""
    import ctypes

    L = F.lib()
    rng = np.random.default_rng(3)
    for n in (0, 1, 1000, 3 * 2 ** 20 + 7):
        src = rng.integers(0, 255, n + 3, dtype=np.uint8)
        dst = np.zeros(n + 3, dtype=np.uint8)
        assert L.fmv_host_copy(dst.ctypes.data + 3, src.ctypes.data + 1, n) == 0
        assert np.array_equal(dst[3:], src[1:n + 1])
        assert not dst[:3].any()
    assert L.fmv_host_copy(None, ctypes.c_void_p(src.ctypes.data), 16) == 1  # FMV_EINVAL
    assert L.fmv_host_copy(None, None, 0) == 0


def test_precision_config_grammar():
    c = F.parse_precision_config("dssdd")
    assert c.render() == "dssdd" and c[1] == F.Precision.Single and c[0] == F.Precision.Double
    for bad, pos in (("dsxdd", 3), ("Dssdd", 1), ("dsshd", 4)):
        with pytest.raises(ValueError, match=f"position {pos}"):
            F.parse_precision_config(bad)
    with pytest.raises(ValueError, match="exactly 5"):
        F.parse_precision_config("dss")
    allc = [c.render() for c in F.enumerate_configs()]
    assert len(allc) == 32 and len(set(allc)) == 32 and allc == sorted(allc)
    assert allc[0] == "ddddd" and allc[-1] == "sssss"
    assert all(F.parse_precision_config(s).render() == s for s in allc)
    ext = [c.render() for c in F.enumerate_configs(include_half=True)]
    assert ext[:32] == allc and "ddhdd" in ext and "hdhdh" in ext and len(ext) == 3 * 2 * 4 * 2 * 3
    # 'm' (fp32 storage, fp64 accumulation) exists at the SBGEMV slot only
    assert "ddmdd" in ext and "sdmsh" in ext and not any("m" in c[:2] + c[3:] for c in ext)
    c = F.parse_precision_config("ddmdd")
    assert c[2] == F.Precision.SingleAccDouble and c.render() == "ddmdd"
    for bad, pos in (("mdddd", 1), ("dmddd", 2), ("dddmd", 4), ("ddddm", 5)):
        with pytest.raises(ValueError, match=f"position {pos}"):
            F.parse_precision_config(bad)
    with pytest.raises(ValueError, match="position 3"):
        F.parse_precision_config("ddmdd", allow_half=False)


def test_dims_and_block_vectors():
    d = F.ProblemDims(5, 3, 7)
    assert d.fft_len() == 14 and d.n_bins() == 8
    with pytest.raises(ValueError):
        F.ProblemDims(0, 1, 1)
    v = F.BlockVector.time_double(3, 4, np.arange(12.0))
    t = F.reorder(v, F.Layout.TOSI)
    assert t.layout == F.Layout.TOSI and t.data[1] == 4.0
    assert np.array_equal(F.reorder(t, F.Layout.SOTI).data, v.data)  # involution, bitwise
    with pytest.raises(ValueError):
        F.BlockVector.time_double(3, 4, np.arange(11.0))
    with pytest.raises(ValueError):
        F.BlockColumn(d, np.zeros(5))


def test_gemv_host_helpers():
    assert F.effective_bandwidth(128, 4096, 100, 4, 1.0) == pytest.approx(0.2114048, rel=1e-12)
    assert F.effective_bandwidth(1, 1, 1, 8, 1.0) == pytest.approx(2.4e-8)
    with pytest.raises(ValueError):
        F.effective_bandwidth(1, 1, 1, 8, 0.0)
    T = F.TilingParams(dispatch_ratio=0.25)
    assert F.select_kernel(100, 5000, F.GemvMode.ConjTrans, T) == F.KernelChoice.Tiled
    assert F.select_kernel(4096, 4096, F.GemvMode.Trans, T) == F.KernelChoice.Naive
    assert F.select_kernel(100, 5000, F.GemvMode.NoTrans, T) == F.KernelChoice.Naive


def test_grid_tree_reduce_and_sharding(orc):
    g = golden("partition")
    assert F.Grid1xP.split(3, 5).shard_ranges == [tuple(r) for r in g["grid_3_5"]]
    assert F.Grid1xP.split(2, 4).shard_ranges == [(0, 2), (2, 4)]
    with pytest.raises(ValueError):
        F.Grid1xP.split(6, 5)
    bufs = list(g["tree_in"])
    assert np.array_equal(F.tree_reduce(bufs, F.Precision.Double), g["tree_d"])
    assert np.array_equal(F.tree_reduce(bufs, F.Precision.Single), g["tree_s"])
    assert np.array_equal(F.tree_reduce([np.full(3, v) for v in (1.0, 2.0, 3.0, 4.0)], F.Precision.Double), [10.0] * 3)
    dims = F.ProblemDims(5, 3, 4)
    col = F.BlockColumn(dims, np.arange(60.0))
    shards = F.shard_operator(col, F.Grid1xP.split(3, 5))
    blocks = np.concatenate([s.data.reshape(4, -1) for s in shards], axis=1).reshape(-1)
    assert np.array_equal(blocks, col.data)  # concatenation reconstructs the column bitwise
    cs = F.CommSpec.forward_reduce(F.parse_precision_config("dddds"), dims)
    assert cs.precision == F.Precision.Single and cs.buffer_len == 12


def test_pareto_and_optimal_bruteforce():
    rng = np.random.default_rng(7)
    cfgs = F.enumerate_configs()
    for trial in range(200):
        n = int(rng.integers(1, 33))
        rows = [F.ConfigResult(cfgs[i], float(rng.integers(1, 6)), 0, 0, float(rng.integers(0, 5)) * 1e-8)
                for i in range(n)]
        front = F.pareto_front(rows)
        brute = [r for r in rows if not any((q.mean_s <= r.mean_s and q.rel_error <= r.rel_error and
                                             (q.mean_s < r.mean_s or q.rel_error < r.rel_error)) for q in rows)]
        assert front == brute
        tol = 2.5e-8
        ok = [r for r in rows if r.rel_error <= tol]
        if not ok:
            with pytest.raises(ValueError):
                F.optimal_config(rows, tol)
            continue
        best = min(ok, key=lambda r: (r.mean_s, r.rel_error, r.config.render()))
        got = F.optimal_config(rows, tol)
        assert got == best.config
        assert any(r.config == got for r in front)  # the constrained optimum lies on the front


def test_pareto_matches_reference(ref):
    rng = np.random.default_rng(8)
    cfgs = [c.render() for c in F.enumerate_configs()]
    for _ in range(50):
        means = rng.integers(1, 5, 32).astype(float)
        errs = rng.integers(0, 4, 32) * 1e-7
        rows = [F.ConfigResult(F.parse_precision_config(c), m, m, m, e) for c, m, e in zip(cfgs, means, errs)]
        mask = ref.pareto(means, errs, cfgs)
        assert [r.config.render() for r in F.pareto_front(rows)] == [c for c, k in zip(cfgs, mask) if k]
        assert F.optimal_config(rows, 1.5e-7).render() == ref.optimal(means, errs, cfgs, 1.5e-7)


def test_sweep_csv_json_roundtrip():
    cfgs = F.enumerate_configs()
    rows = [F.ConfigResult(c, 1.0 + i, 0.5 + i, 2.0 + i, 0.0 if i == 0 else 1e-9 * i) for i, c in enumerate(cfgs)]
    rep = F.make_report(F.ProblemDims(500, 20, 200), F.MatvecKind.Forward, 10, 1e-7, rows)
    back = F.parse_sweep_csv(rep and F.to_csv(rep))
    assert [(r.config, r.mean_s, r.min_s, r.max_s, r.rel_error) for r in back] == \
           [(r.config, r.mean_s, r.min_s, r.max_s, r.rel_error) for r in rows]
    j = F.to_json(rep)
    assert j["kind"] == "forward" and len(j["rows"]) == 32 and j["chosen"] == rep.chosen.render()
    assert F.parse_sweep_csv("# comment\nddddd,1,1,1,0\n")[0].mean_s == 1.0
    with pytest.raises(ValueError, match="missing"):
        F.parse_sweep_csv("ddddd,1,1\n")


def test_cpp_dropin_host_checks():
    exe = os.path.join(ROOT, "build", "fftmv_cpp_tests")
    if not os.path.exists(exe):
        pytest.skip("build/fftmv_cpp_tests not built (make cpp)")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
