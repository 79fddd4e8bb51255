"""Small cases for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_10202_b200 as F
nm, nd, nt = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else (50, 10, 20)
cfgs = sys.argv[4].split(",") if len(sys.argv) > 4 else ["ddddd"]
col = F.uniform_fill(nm * nd * nt, 1)
op = F.setup_operator(F.BlockColumn(F.ProblemDims(nm, nd, nt), col))
for cfg in cfgs:
    f = F.forward_matvec(op, F.uniform_fill(nm * nt, 2), cfg).output.data
    a = F.adjoint_matvec(op, F.uniform_fill(nd * nt, 3), cfg).output.data
    print(cfg, "ok", float(np.abs(f).sum()), float(np.abs(a).sum()))
# block (multi-RHS) matvec over the same operator: FMV_SAN_BLOCK=K
K = int(os.environ.get("FMV_SAN_BLOCK", "0"))
if K:
    for cfg in cfgs:
        B = F.forward_matvec_block(op, np.stack([F.uniform_fill(nm * nt, 10 + r) for r in range(K)]), cfg)
        A = F.adjoint_matvec_block(op, np.stack([F.uniform_fill(nd * nt, 20 + r) for r in range(K)]), cfg)
        print("block", K, cfg, "ok", float(np.abs(B).sum()), float(np.abs(A).sum()))
