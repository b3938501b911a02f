"""Small invocation of every device entry point, for compute-sanitizer
(memcheck / racecheck / synccheck) runs: python tools/sanitize_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import _native as N

n = int(os.environ.get("PROBE_N", "131072"))
d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 1)
inst = P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
h = N.handle()
for engine in (1, 2):  # TMA engine, warp-segment engine
    h.lib.cqk_set_engine(h.ptr, engine)
    for fix in (True, False):
        out = P.solve_cqk(inst, P.SolverOptions(variable_fixing=fix))
        assert out.status is P.Status.SOLVED
h.lib.cqk_set_engine(h.ptr, 0)
P.jacobi_solve(inst)
P.eval_phi(inst, 1.0)
P.eval_x(inst, 1.0, idx=np.arange(0, n, 3))
P.initial_multiplier(inst)
y = P.gen_simplex_y("simplex-n01", n, 2)
P.newton_project_simplex(y, 1.0)
P.newton_project_simplex(y, 1.0, start="alg2")
P.project_l1(y, 1.0)
Y = y[: 64 * 1024].reshape(64, 1024)
P.project_simplex_rows(Y, 1.0)
print("probe ok")

# the large-n routes at probe sizes: run with CQK_FUSED_MIN_N=0
# CQK_SPX_CAPTURE_MIN_N=0 CQK_FUSED_GUESS=2 (forced guess) to sanitize the fused
# start, the direction guess, the capture start, the sparse final and the sparse output
if os.environ.get("PROBE_LARGE_ROUTES"):
    import torch

    P.simplex.SPARSE_MIN_N = 0
    out = P.solve_cqk(inst)
    ref = P.solve_cqk(inst, P.SolverOptions(compact_ratio=2.0))
    assert out.status is P.Status.SOLVED and abs(out.lam - ref.lam) <= 1e-12 * max(1.0, abs(ref.lam))
    yd = torch.from_numpy(y).cuda()
    for l1 in (False, True):
        x = P.project_l1(yd, 1.0) if l1 else P.newton_project_simplex(yd, 1.0).x
        idx, val = P.project_l1(yd, 1.0, output="sparse") if l1 else \
            P.newton_project_simplex(yd, 1.0, output="sparse").sparse
        assert torch.equal(idx, torch.nonzero(x != 0).flatten())
    print("large routes ok")
