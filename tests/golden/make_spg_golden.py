"""SPG fixtures from the REAL reference (cqksolve/spg.py): inputs and the
reference's results for an SVM dual and a basis-pursuit run, so the GPU tests
can compare the device-resident driver with the reference on the same data.

  PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_spg_golden.py
"""
import os

import numpy as np
from cqksolve import build_basis_pursuit, build_svm_dual, spg_solve
from cqksolve.instances import gen_blobs, gen_sparse_ls

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spg.npz")
pts, labels = gen_blobs(80, 20, 3.0, 3)
svm = spg_solve(build_svm_dual(pts, labels, gamma=0.05, C=1.0), np.zeros(80), tol=1e-4)
A, b, xt = gen_sparse_ls(200, 1000, 0.02, 10, 0)
A = A.toarray()
radius = float(np.abs(xt).sum())
bp = {}
for warm in (False, True):
    bp[warm] = spg_solve(build_basis_pursuit(A, b, radius=radius, warm_start=warm),
                         np.zeros(1000), tol=1e-4, max_iter=5000)
np.savez_compressed(
    OUT, pts=pts, labels=labels, svm_x=svm.x, svm_it=svm.iterations, svm_conv=svm.converged,
    svm_obj=svm.objectives[-1], A=A, b=b, radius=radius,
    bp_cold_x=bp[False].x, bp_cold_it=bp[False].iterations, bp_cold_obj=bp[False].objectives[-1],
    bp_cold_inner=np.array([c for c, _ in bp[False].inner_iterations]),
    bp_warm_x=bp[True].x, bp_warm_it=bp[True].iterations, bp_warm_obj=bp[True].objectives[-1],
    bp_warm_inner=np.array([c for c, _ in bp[True].inner_iterations]))
print("svm", svm.iterations, svm.converged, "bp cold", bp[False].iterations, "warm", bp[True].iterations)
