"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the C oracle.

The oracle is a CPU restatement of the reference `cqksolve` hot path
(see cqk_oracle.h for the file:line map).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg may import this module; the product package
never does.
"""

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "libcqk_oracle.so")

SOLVED, INFEASIBLE, E_DOMAIN, E_MAXITER, E_CONTRACT = 0, 1, -1, -2, -3
FIELDS = ("d", "a", "b", "l", "u", "r", "bounds", "y", "xbar")
TAU64 = float(np.finfo(np.float64).eps) ** 0.75


class Result(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("domain_field", ctypes.c_int32),
        ("domain_index", ctypes.c_int64),
        ("lam", ctypes.c_double),
        ("lam0", ctypes.c_double),
        ("iterations", ctypes.c_int64),
        ("phi_evals", ctypes.c_int64),
        ("fixed_count", ctypes.c_int64),
        ("bracket_lo", ctypes.c_double),
        ("bracket_hi", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def build(force=False):
    """Compile the oracle with its Makefile (gcc, OpenMP)."""
    srcs = ("cqk_oracle.c", "cqk_gen.c", "cqk_oracle.h")
    if force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(_HERE, f)) for f in srcs
    ):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return LIB_PATH


_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_U8 = ctypes.POINTER(ctypes.c_uint8)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        dbl, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        R = ctypes.POINTER(Result)
        L.orc_pairwise_sum.argtypes = [_D, i64]
        L.orc_pairwise_sum.restype = dbl
        L.orc_validate.argtypes = [_D] * 5 + [i64, dbl, R]
        L.orc_initial_multiplier.argtypes = [_D] * 5 + [i64, dbl, _D]
        L.orc_initial_multiplier.restype = dbl
        L.orc_phi_scan.argtypes = [_D] * 5 + [_I64, i64, dbl, _D, _U8, _U8]
        L.orc_eval_x.argtypes = [_D] * 5 + [_I64, i64, dbl, _D]
        L.orc_secant_step.argtypes = [dbl] * 5 + [_D]
        L.orc_nearest_breakpoint.argtypes = [_D] * 5 + [_I64, i64, dbl, i32, _D]
        L.orc_solve_cqk.argtypes = [_D] * 5 + [i64, dbl, i32, i64, dbl, _D, dbl, i32, _D, R]
        L.orc_jacobi_solve.argtypes = [_D] * 5 + [i64, dbl, i64, dbl, i32, dbl, i32, _D, R]
        L.orc_par_solve_cqk.argtypes = [_D] * 5 + [i64, dbl, i32, i64, dbl, i32, _D, i64,
                                                   dbl, i32, _D, R]
        L.orc_simplex_init_lambda.argtypes = [_D, i64, dbl, _I64, i64, _D, i32, _D, _I64,
                                              _I64, _U8, _D]
        L.orc_newton_project_simplex.argtypes = [_D, i64, dbl, i32, i64, dbl, _D, i32, dbl,
                                                 _D, _D, i64, R]
        L.orc_project_l1.argtypes = [_D, i64, dbl, i32, i64, dbl, _D, _D, R]
        L.orc_par_simplex_init.argtypes = [_D, i64, dbl, i32, _D, _I64, _I64, _U8, _D]
        L.orc_newton_simplex_from.argtypes = [_D, i64, dbl, i32, i64, dbl, dbl, _I64, i64, _D, R]
        L.orc_exact_simplex_lambda.argtypes = [_D, i64, dbl]
        L.orc_exact_simplex_lambda.restype = dbl
        L.orc_project_simplex_rows.argtypes = [_D, i64, i64, dbl, i32, _D, _D, _I64]
        L.orc_project_simplex_rows.restype = i64
        L.orc_gen_cqk.argtypes = [i32, i64, ctypes.c_uint64] + [_D] * 6
        L.orc_gen_simplex_y.argtypes = [i32, i64, ctypes.c_uint64, _D]
        _lib = L
    return _lib


def _p(arr, kind=_D):
    if arr is None:
        return None
    return arr.ctypes.data_as(kind)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _arrays(d, a, b, l, u):
    return [_f64(v) for v in (d, a, b, l, u)]


def pairwise_sum(a):
    a = _f64(a)
    return lib().orc_pairwise_sum(_p(a), a.size)


def validate(d, a, b, l, u, r):
    arrs = _arrays(d, a, b, l, u)
    res = Result()
    st = lib().orc_validate(*[_p(v) for v in arrs], arrs[0].size, float(r), ctypes.byref(res))
    if st == 0:
        return None
    idx = res.domain_index if res.domain_index >= 0 else None
    return FIELDS[res.domain_field], idx


def initial_multiplier(d, a, b, l, u, r, xbar=None):
    arrs = _arrays(d, a, b, l, u)
    xb = None if xbar is None else _f64(xbar)
    return lib().orc_initial_multiplier(*[_p(v) for v in arrs], arrs[0].size, float(r), _p(xb))


def phi_scan(d, a, b, l, u, lam, idx=None):
    """core.py:182 _phi_scan -> (value, dminus, dplus, abs_bx, at_lower, at_upper)."""
    arrs = _arrays(d, a, b, l, u)
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    m = arrs[0].size if ix is None else ix.size
    out = np.zeros(4)
    lo = np.zeros(m, np.uint8)
    hi = np.zeros(m, np.uint8)
    lib().orc_phi_scan(*[_p(v) for v in arrs], _p(ix, _I64), m, float(lam), _p(out),
                       _p(lo, _U8), _p(hi, _U8))
    return (float(out[0]), float(out[1]), float(out[2]), float(out[3]),
            lo.astype(bool), hi.astype(bool))


def eval_x(d, a, b, l, u, lam, idx=None):
    arrs = _arrays(d, a, b, l, u)
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    m = arrs[0].size if ix is None else ix.size
    x = np.empty(m)
    lib().orc_eval_x(*[_p(v) for v in arrs], _p(ix, _I64), m, float(lam), _p(x))
    return x


def secant_step(lo, phi_lo, hi, phi_hi, r):
    out = ctypes.c_double()
    st = lib().orc_secant_step(lo, phi_lo, hi, phi_hi, r, ctypes.byref(out))
    if st:
        raise ArithmeticError("invalid secant bracket")
    return out.value


def nearest_breakpoint(d, a, b, l, u, edge, right, idx=None):
    arrs = _arrays(d, a, b, l, u)
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    m = arrs[0].size if ix is None else ix.size
    out = ctypes.c_double()
    found = lib().orc_nearest_breakpoint(*[_p(v) for v in arrs], _p(ix, _I64), m, float(edge),
                                         0 if right else 1, ctypes.byref(out))
    return out.value if found else None


def _finish(st, res, x):
    out = res.as_dict()
    out["status"] = st
    out["x"] = x if st == SOLVED else None
    return out


def solve_cqk(d, a, b, l, u, r, fixing=True, max_iter=100, tau=TAU64, xbar=None,
              lam0=None, check=True, want_x=True):
    arrs = _arrays(d, a, b, l, u)
    n = arrs[0].size
    x = np.empty(n) if want_x else None
    xb = None if xbar is None else _f64(xbar)
    res = Result()
    st = lib().orc_solve_cqk(*[_p(v) for v in arrs], n, float(r), int(fixing), int(max_iter),
                             float(tau), _p(xb), math.nan if lam0 is None else float(lam0),
                             int(check), _p(x), ctypes.byref(res))
    return _finish(st, res, x)


def jacobi_solve(d, a, b, l, u, r, workers=1, max_iter=100, tau=TAU64, lam0=None,
                 check=True, want_x=True):
    arrs = _arrays(d, a, b, l, u)
    n = arrs[0].size
    x = np.empty(n) if want_x else None
    res = Result()
    st = lib().orc_jacobi_solve(*[_p(v) for v in arrs], n, float(r), int(max_iter), float(tau),
                                int(workers), math.nan if lam0 is None else float(lam0),
                                int(check), _p(x), ctypes.byref(res))
    return _finish(st, res, x)


def par_solve_cqk(d, a, b, l, u, r, workers=1, fixing=True, max_iter=100, tau=TAU64,
                  xbar=None, merge_threshold=1024, lam0=None, check=True, want_x=True):
    arrs = _arrays(d, a, b, l, u)
    n = arrs[0].size
    x = np.empty(n) if want_x else None
    xb = None if xbar is None else _f64(xbar)
    res = Result()
    st = lib().orc_par_solve_cqk(*[_p(v) for v in arrs], n, float(r), int(fixing), int(max_iter),
                                 float(tau), int(workers), _p(xb), int(merge_threshold),
                                 math.nan if lam0 is None else float(lam0), int(check), _p(x),
                                 ctypes.byref(res))
    return _finish(st, res, x)


def simplex_init_lambda(y, r, xbar=None, sharpened=False):
    y = _f64(y)
    n = y.size
    J = np.empty(n, np.int64)
    nJ = ctypes.c_int64()
    fixed = np.zeros(n, np.uint8)
    lam = ctypes.c_double()
    sJ = ctypes.c_double()
    xb = None if xbar is None else _f64(xbar)
    lib().orc_simplex_init_lambda(_p(y), n, float(r), None, n, _p(xb), int(sharpened),
                                  ctypes.byref(lam), _p(J, _I64), ctypes.byref(nJ),
                                  _p(fixed, _U8), ctypes.byref(sJ))
    return lam.value, J[:nJ.value].copy(), fixed.astype(bool), sJ.value


def newton_project_simplex(y, r, fixing=True, max_iter=100, tau=TAU64, xbar=None,
                           sharpened=False, lam0=None, want_x=True, trace=False):
    y = _f64(y)
    n = y.size
    x = np.empty(n) if want_x else None
    cap = 4096 if trace else 0
    tr = np.zeros((cap, 4)) if trace else None
    xb = None if xbar is None else _f64(xbar)
    res = Result()
    st = lib().orc_newton_project_simplex(_p(y), n, float(r), int(fixing), int(max_iter),
                                          float(tau), _p(xb), int(sharpened),
                                          math.nan if lam0 is None else float(lam0), _p(x),
                                          _p(tr), cap, ctypes.byref(res))
    out = _finish(st, res, x)
    if trace:
        out["trace"] = [tuple(row) for row in tr[: min(res.phi_evals, cap)]]
    return out


def project_l1(y, r, fixing=True, max_iter=100, tau=TAU64, xbar=None):
    y = _f64(y)
    n = y.size
    x = np.empty(n)
    xb = None if xbar is None else _f64(xbar)
    res = Result()
    st = lib().orc_project_l1(_p(y), n, float(r), int(fixing), int(max_iter), float(tau), _p(xb),
                              _p(x), ctypes.byref(res))
    return _finish(st, res, x)


def exact_simplex_lambda(y, r):
    y = _f64(y)
    return lib().orc_exact_simplex_lambda(_p(y), y.size, float(r))


def par_simplex_init(y, r, workers=1):
    """parallel.py:330-368 -> (lambda0, free, fixed_mask, sum_free)."""
    y = _f64(y)
    n = y.size
    free = np.empty(n, np.int64)
    nf = ctypes.c_int64()
    fixed = np.zeros(n, np.uint8)
    lam = ctypes.c_double()
    sj = ctypes.c_double()
    lib().orc_par_simplex_init(_p(y), n, float(r), int(workers), ctypes.byref(lam), _p(free, _I64),
                               ctypes.byref(nf), _p(fixed, _U8), ctypes.byref(sj))
    return lam.value, free[: nf.value].copy(), fixed.astype(bool), sj.value


def newton_simplex_from(y, r, lam0, free, fixing=True, max_iter=100, tau=TAU64, want_x=True):
    """Algorithm 4 from (lam0, free set) without the lambda0= clamp."""
    y = _f64(y)
    f = np.ascontiguousarray(free, dtype=np.int64)
    x = np.empty(y.size) if want_x else None
    res = Result()
    st = lib().orc_newton_simplex_from(_p(y), y.size, float(r), int(fixing), int(max_iter),
                                       float(tau), float(lam0), _p(f, _I64), f.size, _p(x),
                                       ctypes.byref(res))
    return _finish(st, res, x)


def project_simplex_rows(Y, r, threads=1, want_x=True):
    """newton_project_simplex per row (OpenMP over rows) -> (X, lam, iterations, failed)."""
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    rows, cols = Y.shape
    X = np.empty_like(Y) if want_x else None
    lam = np.empty(rows)
    its = np.empty(rows, np.int64)
    bad = lib().orc_project_simplex_rows(_p(Y), rows, cols, float(r), int(threads), _p(X), _p(lam),
                                         _p(its, _I64))
    return X, lam, its, int(bad)


CQK_FAMILIES = ("cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated")
SIMPLEX_FAMILIES = ("simplex-u01", "simplex-n01", "simplex-n0m3")


def gen_cqk(family, n, seed):
    """instances.py:43-70 (cqk_gen.c): (d, a, b, l, u, r), r from pairwise dots."""
    arrs = [np.empty(int(n)) for _ in range(5)]
    r = ctypes.c_double()
    rc = lib().orc_gen_cqk(CQK_FAMILIES.index(family), int(n), int(seed) & (2**64 - 1),
                           *[_p(v) for v in arrs], ctypes.byref(r))
    if rc != 0:
        raise ValueError(f"orc_gen_cqk failed ({rc})")
    return (*arrs, r.value)


def gen_simplex_y(family, n, seed):
    """instances.py:73-86 (cqk_gen.c)."""
    y = np.empty(int(n))
    rc = lib().orc_gen_simplex_y(SIMPLEX_FAMILIES.index(family), int(n), int(seed) & (2**64 - 1),
                                 _p(y))
    if rc != 0:
        raise ValueError(f"orc_gen_simplex_y failed ({rc})")
    return y


def exact_lambda(d, a, b, l, u, r):
    """Exact root of phi(lam) = r by bisection over the sorted breakpoints and
    one interpolation on the bracketing affine piece (the method of the
    reference's oracle.py:23-85, restated) -> (status, lam or None).  Plain
    numpy, O(n log n): a check for small and medium n."""
    d, a, b, l, u = (np.asarray(v, dtype=np.float64) for v in (d, a, b, l, u))
    r = float(r)

    def phi(lam):
        return float(b @ np.clip((b * lam + a) / d, l, u))

    fl, fu = np.isfinite(l), np.isfinite(u)
    bps = np.unique(np.concatenate([(d[fl] * l[fl] - a[fl]) / b[fl], (d[fu] * u[fu] - a[fu]) / b[fu]]))
    w = b * b / d
    if bps.size == 0:
        return SOLVED, (r - float(b @ (a / d))) / float(w.sum())
    top, bot = phi(bps[-1]), phi(bps[0])
    if r > top:
        s = float(w[u == np.inf].sum())
        return (INFEASIBLE, None) if s == 0.0 else (SOLVED, bps[-1] + (r - top) / s)
    if r < bot:
        s = float(w[l == -np.inf].sum())
        return (INFEASIBLE, None) if s == 0.0 else (SOLVED, bps[0] - (bot - r) / s)
    lo, hi = 0, bps.size - 1  # phi(bps[hi]) >= r > phi(bps[lo - 1])
    if bot >= r:
        hi = 0
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if phi(bps[mid]) >= r:
            hi = mid
        else:
            lo = mid
    vh = phi(bps[hi])
    if vh == r:  # on a plateau: its left end
        while hi > 0 and phi(bps[hi - 1]) == r:
            hi -= 1
        return SOLVED, float(bps[hi])
    vl = phi(bps[hi - 1])
    return SOLVED, float(bps[hi - 1] + (r - vl) * (bps[hi] - bps[hi - 1]) / (vh - vl))
