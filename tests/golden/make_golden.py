"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/libfftmv_ref.so: /root/reference/proj/include compiled verbatim,
FFTW API served by MKL DFTI). Run in the dev container, where /root/reference
exists:  python tests/golden/make_golden.py

Inputs are not stored: they are regenerated from seeds with the reference
fills (random_fill.hpp), whose outputs are themselves pinned in fills.npz.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("MKL_NUM_THREADS", "1")

from oracle.oracle import ref  # noqa: E402

S = 20250814
R = ref()


def inputs(nm, nd, nt, fill="uni", seed=S):
    if fill == "uni":
        f = lambda n, k: R.uniform_fill(n, R.seed_stream(seed, k))  # noqa: E731
    else:
        f = lambda n, k: R.non_representable_fill(n, R.seed_stream(seed, k))  # noqa: E731
    return f(nm * nd * nt, 0), f(nm * nt, 1), f(nd * nt, 2)


def configs():
    out = []
    for bits in range(32):
        out.append("".join("s" if (bits >> (4 - i)) & 1 else "d" for i in range(5)))
    return out


def main():
    g = {}
    # ---- fills (random_fill.hpp:17-32, sweep.hpp:32-46)
    g["fill_uniform_seed7"] = R.uniform_fill(64, 7)
    g["fill_uniform_seed7_0_5"] = R.uniform_fill(64, 7, 0.0, 5.0)
    g["fill_nonrep_seed9"] = R.non_representable_fill(64, 9)
    g["seed_stream"] = np.array([R.seed_stream(S, k) for k in range(4)], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "fills.npz"), **g)

    # ---- FFT (fft.hpp:110-148), SPEC.md:118-134 examples
    f = {}
    f["ones8"] = R.fft_forward(8, 1, np.ones(8))
    delta = np.zeros(8)
    delta[0] = 1
    f["delta8"] = R.fft_forward(8, 1, delta)
    x16 = R.uniform_fill(16, 11)
    f["rand16_in"] = x16
    f["rand16"] = R.fft_forward(16, 1, x16)
    x400 = R.uniform_fill(3 * 400, 12)
    f["rand400x3_in"] = x400
    f["rand400x3"] = R.fft_forward(400, 3, x400)
    f["rand400x3_f32"] = R.fft_forward(400, 3, x400.astype(np.float32), prec=0)
    f["inv400x3"] = R.fft_inverse(400, 3, f["rand400x3"])
    f["inv400x3_f32"] = R.fft_inverse(400, 3, f["rand400x3_f32"], prec=0)
    x2000 = R.uniform_fill(2 * 2000, 13)
    f["rand2000x2_in"] = x2000
    f["rand2000x2"] = R.fft_forward(2000, 2, x2000)
    np.savez_compressed(os.path.join(HERE, "fft.npz"), **f)

    # ---- operator setup (operator.hpp:99-125)
    s = {}
    for (nm, nd, nt) in [(3, 2, 4), (16, 4, 32), (5, 3, 7)]:
        col, _, _ = inputs(nm, nd, nt)
        s[f"bins_{nm}_{nd}_{nt}"] = R.setup_operator(nm, nd, nt, col).bins()
    np.savez_compressed(os.path.join(HERE, "setup.npz"), **s)

    # ---- matvecs (matvec.hpp:233-318): all 32 configs at 16/4/32, three at C1
    mv = {}
    for fill in ("uni", "nonrep"):
        nm, nd, nt = 16, 4, 32
        col, m, d = inputs(nm, nd, nt, fill)
        op = R.setup_operator(nm, nd, nt, col)
        for cfg in configs():
            mv[f"{fill}_16_4_32_F_{cfg}"] = R.matvec(op, 0, cfg, m)
            mv[f"{fill}_16_4_32_A_{cfg}"] = R.matvec(op, 1, cfg, d)
        mv[f"{fill}_16_4_32_dense_F"] = R.dense(0, nm, nd, nt, col, m)
        mv[f"{fill}_16_4_32_dense_A"] = R.dense(1, nm, nd, nt, col, d)
    nm, nd, nt = 100, 10, 100
    for fill in ("uni", "nonrep"):
        col, m, d = inputs(nm, nd, nt, fill)
        op = R.setup_operator(nm, nd, nt, col)
        r0f, r0a = R.matvec(op, 0, "ddddd", m), R.matvec(op, 1, "ddddd", d)
        errs = np.zeros((32, 2))
        casts = np.zeros(32, dtype=np.int64)
        for i, cfg in enumerate(configs()):
            R.reset_casts()
            rf = R.matvec(op, 0, cfg, m)
            casts[i] = R.casts()
            ra = R.matvec(op, 1, cfg, d)
            errs[i, 0] = np.linalg.norm(rf - r0f) / np.linalg.norm(r0f)
            errs[i, 1] = np.linalg.norm(ra - r0a) / np.linalg.norm(r0a)
            if cfg in ("ddddd", "dssdd", "sssss"):
                mv[f"{fill}_C1_F_{cfg}"] = rf
                mv[f"{fill}_C1_A_{cfg}"] = ra
        mv[f"{fill}_C1_errors"] = errs
        mv[f"{fill}_C1_casts_forward"] = casts
    np.savez_compressed(os.path.join(HERE, "matvec.npz"), **mv)

    # ---- GEMV (gemv.hpp:135-201) naive outputs
    gm = {}
    rng = np.random.default_rng(5)
    for dt in ("s", "d", "c", "z"):
        npdt = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}[dt]
        for mode in (0, 1, 2):
            m_, n_, b_ = 7, 13, 3
            A = rng.standard_normal(m_ * n_ * b_).astype(npdt)
            xl, yl = (n_, m_) if mode == 0 else (m_, n_)
            x = rng.standard_normal(xl * b_).astype(npdt)
            if dt in "cz":
                A = A + 1j * rng.standard_normal(A.size).astype(A.real.dtype)
                x = x + 1j * rng.standard_normal(x.size).astype(x.real.dtype)
                A, x = A.astype(npdt), x.astype(npdt)
            y = np.zeros(yl * b_, dtype=npdt)
            R.gemv(0, mode, dt, m_, n_, b_, m_, m_ * n_, A, xl, x, yl, y)
            gm[f"{dt}{mode}_A"], gm[f"{dt}{mode}_x"], gm[f"{dt}{mode}_y"] = A, x, y
    np.savez_compressed(os.path.join(HERE, "gemv.npz"), **gm)

    # ---- partition (partition.hpp:84-217), acceptance 8 shape 64/4/32
    pt = {}
    nm, nd, nt = 64, 4, 32
    col, m, d = inputs(nm, nd, nt)
    for p in (1, 2, 4, 8, 16):
        for cfg in ("ddddd", "dddds", "sdddd"):
            pt[f"p{p}_F_{cfg}"] = R.matvec_partitioned(nm, nd, nt, col, p, 0, cfg, m)
            pt[f"p{p}_A_{cfg}"] = R.matvec_partitioned(nm, nd, nt, col, p, 1, cfg, d)
    pt["grid_3_5"] = np.array(R.grid_split(3, 5))
    bufs = [R.uniform_fill(10, 40 + k) for k in range(7)]
    pt["tree_in"] = np.stack(bufs)
    pt["tree_d"] = R.tree_reduce(bufs, True)
    pt["tree_s"] = R.tree_reduce(bufs, False)
    np.savez_compressed(os.path.join(HERE, "partition.npz"), **pt)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
