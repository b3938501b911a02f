"""Data-parallel drivers (drop-in for cqksolve.parallel, parallel.py:1-500).

On the B200 the "workers" of the reference's thread pool are the SMs of the
device: jacobi_solve and par_solve_cqk run the same single persistent kernel
as solve_cqk with the respective driver's decision logic (fixing-free
Jacobi, parallel.py:371-500; chunked fixing, parallel.py:174-327).  The
`workers` argument is accepted for signature compatibility; the degree of
parallelism is the full GPU.  Multi-GPU sharding lives in `distributed.py`.
"""

import os

from . import _native as N
from .newton import SolverOptions, run_cqk

__all__ = ["par_solve_cqk", "jacobi_solve", "resolve_workers", "MERGE_THRESHOLD"]

MERGE_THRESHOLD = 1024


def resolve_workers(workers=None):
    """Explicit argument beats CQK_WORKERS (parallel.py:52-59)."""
    if workers is not None:
        return max(1, int(workers))
    env = os.environ.get("CQK_WORKERS")
    if env:
        return max(1, int(env))
    return 1


def _tree_sum(values):
    """The determinism contract of the reference's chunk reductions
    (parallel.py:62-72): adjacent pairs summed level by level, an odd tail
    carried up unchanged.  The device reductions across CTAs and ranks use
    fixed orders of the same kind, so reruns are bit-identical; this host
    form serves callers that combine per-device partials themselves."""
    level = list(values)
    if not level:
        raise ValueError("_tree_sum of nothing")
    while len(level) > 1:
        paired = [level[k] + level[k + 1] for k in range(0, len(level) - 1, 2)]
        if len(level) & 1:
            paired.append(level[-1])
        level = paired
    return level[0]


def par_solve_cqk(inst, opts=None, workers=None, xbar=None, check=True,
                  merge_threshold=MERGE_THRESHOLD):
    """Chunked fork-join variant of solve_cqk; same outcome contract (parallel.py:174-327)."""
    resolve_workers(workers)
    return run_cqk(inst, opts, N.VARIANT_PAR, xbar=xbar, check=check)


def jacobi_solve(inst, opts=None, workers=None, check=True):
    """Fixing-free Jacobi variant: stateless maps over all n (parallel.py:371-500)."""
    resolve_workers(workers)
    if opts is None:
        opts = SolverOptions()
    opts = SolverOptions(variable_fixing=False, max_iterations=opts.max_iterations,
                         tolerance_scale=opts.tolerance_scale)
    return run_cqk(inst, opts, N.VARIANT_JACOBI, check=check)
