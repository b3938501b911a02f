"""Safeguarded semismooth Newton solver for the CQK dual equation (drop-in).

Drop-in for cqksolve.newton (/root/reference/pkg/src/cqksolve/newton.py).
`solve_cqk` is ONE persistent cooperative kernel launch on the B200: the
fused validate + lambda0 pass, every phi evaluation with its deterministic
grid reduction, the scalar state machine of newton.py:244-342 (replayed on a
device thread), variable fixing with physical compaction, the rare
breakpoint pass and the final x(lambda*) pass.  The scalar helpers below
(secant_step) and the component-level functions (nearest_breakpoint,
fix_variables) keep the reference's signatures for callers and tests.
"""

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .core import DomainError, Marshal, _is_torch, raise_domain, phi_scan

__all__ = [
    "Status",
    "SolverOptions",
    "SolveState",
    "SolveOutcome",
    "ContractViolation",
    "MaxIterationsError",
    "solve_cqk",
    "secant_step",
    "nearest_breakpoint",
    "fix_variables",
]


class Status(enum.Enum):
    SOLVED = "solved"
    INFEASIBLE = "infeasible"


class ContractViolation(RuntimeError):
    """An internal precondition failed (invalid secant bracket)."""


class MaxIterationsError(RuntimeError):
    """No stopping criterion met within the iteration budget."""

    def __init__(self, message, lam, iterations, phi_evals):
        self.lam = lam
        self.iterations = iterations
        self.phi_evals = phi_evals
        super().__init__(message)


@dataclass
class SolverOptions:
    """Tuning knobs shared by all solver variants (newton.py:52-67).

    tolerance_scale defaults to eps**(3/4) of the instance dtype.
    compact_ratio (B200 only): physically compact the working set when the
    logically fixed share of it reaches this ratio (>1 never).  None = the
    library default: 0.5 on the TMA engine (n >= 64Ki per rank), 0.4 once a
    fused start's guessed survivors were adopted (n >= 8e6 per rank), 0.25 on the
    warp-segment engine (cqk_abi.cu default_compact_ratio).
    """

    variable_fixing: bool = True
    max_iterations: int = 100
    tolerance_scale: float | None = None
    compact_ratio: float | None = None

    def tau(self, dtype):
        if self.tolerance_scale is not None:
            return float(self.tolerance_scale)
        return float(np.finfo(dtype).eps) ** 0.75


@dataclass
class SolveState:
    """Per-solve state (newton.py:70-90); used by the component functions."""

    active: np.ndarray
    r_residual: float
    bracket_lo: float = -np.inf
    bracket_hi: float = np.inf
    lam: float = 0.0
    last_lam: float | None = None
    phi_lo: float | None = None
    phi_hi: float | None = None
    x: np.ndarray | None = None
    fixed_abs: float = 0.0
    fixed_count: int = 0


@dataclass
class SolveOutcome:
    """Result of one solve (newton.py:93-103) plus device statistics."""

    status: Status
    lam: float | None
    x: object
    iterations: int
    phi_evals: int
    fixed_count: int = 0
    sparse: tuple | None = None
    stats: dict = field(default_factory=dict, repr=False, compare=False)


def secant_step(lo, phi_lo, hi, phi_hi, r):
    """Root of the affine interpolant through the bracket (newton.py:106-121)."""
    if not (lo < hi) or not (phi_lo < r < phi_hi):
        raise ContractViolation(
            f"invalid secant bracket: lo={lo}, hi={hi}, phi_lo={phi_lo}, phi_hi={phi_hi}, r={r}")
    lam = lo + (r - phi_lo) * (hi - lo) / (phi_hi - phi_lo)
    if not (lo < lam < hi):
        lam = lo + 0.5 * (hi - lo)
    return lam


class Direction(enum.Enum):
    RIGHT = "right"
    LEFT = "left"


def nearest_breakpoint(state, inst, direction):
    """Closest active breakpoint strictly beyond the bracket edge (newton.py:129-162), on device."""
    m = Marshal(inst.d, inst.a, inst.b, inst.l, inst.u)
    ix, ixp, cnt = m.index(state.active, inst.n)
    h = m.handle()
    right = direction is Direction.RIGHT
    edge = state.bracket_lo if right else state.bracket_hi
    import ctypes

    bp = ctypes.c_double()
    found = ctypes.c_int32()
    rc = h.lib.cqk_nearest_breakpoint_f64(h.ptr, m.mem, *m.ptrs, inst.n, ixp, cnt, float(edge),
                                          1 if right else 0, bp, found)
    if rc != 0:
        raise N.NativeError(f"nearest_breakpoint failed ({rc}): {N.last_error()}")
    return float(bp.value) if found.value else None


def fix_variables(state, inst, lam, phi_value, r, at_lower=None, at_upper=None):
    """Permanently clamp active variables proven to sit at a bound (newton.py:165-206).

    The at-bound masks come from the device scan; the bookkeeping on the
    SolveState (index compaction, residual and bracket shifts) mirrors the
    reference on the host arrays the caller owns."""
    idx = state.active
    if at_lower is None or at_upper is None:
        _, _, _, _, at_lower, at_upper = phi_scan(inst, lam, idx, masks=True)
    to_np = (lambda v: v.cpu().numpy()) if _is_torch(inst.d) else np.asarray
    at_lower = to_np(at_lower)
    at_upper = to_np(at_upper)
    if phi_value > r:
        bound = to_np(inst.l)
        mask = at_lower & np.isfinite(bound[idx])
    elif phi_value < r:
        bound = to_np(inst.u)
        mask = at_upper & np.isfinite(bound[idx])
    else:
        return state
    if not mask.any():
        return state
    newly = idx[mask]
    vals = bound[newly]
    contrib = to_np(inst.b)[newly] * vals
    total = float(contrib.sum())
    state.active = idx[~mask]
    state.r_residual -= total
    state.fixed_abs += float(np.abs(contrib).sum())
    state.fixed_count += newly.size
    if state.x is not None:
        state.x[newly] = vals
    if state.phi_lo is not None:
        state.phi_lo -= total
    if state.phi_hi is not None:
        state.phi_hi -= total
    return state


def _outcome(inst, res, rc, x, what):
    if rc == N.E_DOMAIN:
        raise_domain(res)
    if rc == N.E_MAXITER:
        raise MaxIterationsError(
            f"no stopping criterion met in {int(res.iterations) - 1} iterations (lam={res.lam})",
            lam=float(res.lam), iterations=int(res.iterations), phi_evals=int(res.phi_evals))
    if rc == N.E_CONTRACT:
        raise ContractViolation(f"{what}: invalid secant bracket")
    if rc == N.INFEASIBLE:
        return SolveOutcome(status=Status.INFEASIBLE, lam=None, x=None,
                            iterations=int(res.iterations), phi_evals=int(res.phi_evals),
                            fixed_count=int(res.fixed_count), stats=res.stats())
    if rc != N.SOLVED:
        raise N.NativeError(f"{what} failed ({rc}): {N.last_error()}")
    if x is not None and inst.dtype == np.float32:
        x = x.float() if _is_torch(x) else x.astype(np.float32, copy=False)
    return SolveOutcome(status=Status.SOLVED, lam=float(res.lam), x=x,
                        iterations=int(res.iterations), phi_evals=int(res.phi_evals),
                        fixed_count=int(res.fixed_count), stats=res.stats())


def run_cqk(inst, opts, variant, xbar=None, check=True, lambda0=None, want_x=True, trace=None):
    """Shared driver of solve_cqk / jacobi_solve / par_solve_cqk."""
    if opts is None:
        opts = SolverOptions()
    if xbar is not None:
        shape = tuple(xbar.shape) if hasattr(xbar, "shape") else np.asarray(xbar).shape
        if shape != (inst.n,):
            raise DomainError("xbar", None, "xbar must have length n")
    f32 = inst.dtype == np.float32
    m = Marshal(inst.d, inst.a, inst.b, inst.l, inst.u, xbar, f32=f32)
    h = m.handle()
    x, xp = m.empty(inst.n) if want_x else (None, None)
    o = N.make_options(opts, variant=variant, check=check, lambda0=lambda0,
                       compact_ratio=getattr(opts, "compact_ratio", None),
                       trace=trace is not None,
                       fixing=False if variant == N.VARIANT_JACOBI else None,
                       tau=opts.tau(inst.dtype))
    res = N.Result()
    g = N.env_group() if (m.mem == N.MEM_HOST and trace is None and not f32) else None
    if f32:  # float32 element math (cqk_solve_f32)
        rc = h.lib.cqk_solve_f32(h.ptr, m.mem, *m.ptrs[:5], inst.n, float(inst.r), o, m.ptrs[5],
                                 xp, res)
    elif g is not None:  # CQK_DEVICES: shard the host instance across the group's GPUs
        with g.lock:
            rc = g.lib.cqk_solve_group_f64(g.ptr, *m.ptrs[:5], inst.n, float(inst.r), o, m.ptrs[5],
                                           xp, res)
    else:
        rc = h.lib.cqk_solve_f64(h.ptr, m.mem, *m.ptrs[:5], inst.n, float(inst.r), o, m.ptrs[5],
                                 xp, res)
    if trace is not None:
        trace.extend(h.trace(res.trace_len))
    return _outcome(inst, res, rc, x, "solve_cqk")


def solve_cqk(inst, opts=None, xbar=None, check=True):
    """Solve a CQK instance by the safeguarded semismooth Newton method (newton.py:209-342)."""
    return run_cqk(inst, opts, N.VARIANT_SOLVE, xbar=xbar, check=check)
