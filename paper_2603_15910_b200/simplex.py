"""Projections onto the simplex and the l1 ball (drop-in for cqksolve.simplex).

Device route: the reference's own `lambda0=` route of newton_project_simplex
(simplex.py:246-250) with the start lambda0 = min((r - sum y)/n, r - max y)
(both are upper bounds of the root; "formula" selects the first alone),
followed by Algorithm 4's streamlined Newton iteration with variable fixing
(simplex.py:256-294), all inside one persistent kernel.  The result equals the
reference's Algorithm-2-initialised projection to rounding (the root does not
depend on the start); iteration counts match the reference's `lambda0=` route
with the same start.  A warm start (`xbar`, simplex.py:65-109) -- or
start="alg2" -- runs the reference's Gauss-Seidel initializer per chunk on
the device (par_simplex_init semantics, `sharpened` as given) and Algorithm 4
on its free set.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import DomainError, _is_torch
from .newton import ContractViolation, SolveOutcome, SolverOptions, Status

__all__ = [
    "InitResult",
    "EmptyIndexSet",
    "simplex_init_lambda",
    "par_simplex_init",
    "newton_project_simplex",
    "project_l1",
    "project_simplex_rows",
]


class EmptyIndexSet(ValueError):
    """The candidate index set handed to the initializer is empty."""


@dataclass
class InitResult:
    lambda0: float
    free: np.ndarray
    fixed_mask: np.ndarray
    sum_free: float


def _alg2(y, r, idx, xbar, sharpened, workers):
    import ctypes

    yv, dt, dev = _prep(y)
    n = int(yv.shape[0])
    h = N.handle(yv.get_device() if dev else None)
    import torch

    if dev:
        h.use_current_stream()
        mem = N.MEM_DEVICE
        ix = None if idx is None else torch.as_tensor(idx, device=yv.device).to(torch.int64).contiguous()
        xb = None if xbar is None else xbar.to(torch.float64).contiguous()
        p = n if ix is None else int(ix.numel())
        free = torch.empty(max(p, 1), dtype=torch.int64, device=yv.device)
        fixed = torch.zeros(n, dtype=torch.uint8, device=yv.device)
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        yp = yv.data_ptr()
    else:
        h.use_current_stream()
        mem = N.MEM_HOST
        ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
        xb = None if xbar is None else np.ascontiguousarray(xbar, dtype=np.float64)
        p = n if ix is None else int(ix.size)
        free = np.empty(max(p, 1), np.int64)
        fixed = np.zeros(n, np.uint8)
        ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        yp = yv.ctypes.data
    if p == 0:
        raise EmptyIndexSet("initializer needs at least one candidate index")
    lam, nf, sj, jp = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()
    rc = h.lib.spx_init_alg2_f64(h.ptr, mem, yp, n, float(r), ptr(ix), p, int(workers), ptr(xb),
                                 int(bool(sharpened)), lam, nf, ptr(free), ptr(fixed), sj, jp)
    if rc == N.E_EMPTY:
        raise EmptyIndexSet("initializer needs at least one candidate index")
    if rc != 0:
        raise N.NativeError(f"Algorithm-2 initializer failed ({rc}): {N.last_error()}")
    lam0 = lam.value
    if xbar is not None and jp.value == 0:  # simplex.py:151-152
        y0 = float(yv[0])
        lam0 = max(float(r) / n, -y0)
    fm = fixed.bool() if dev else fixed.astype(bool)
    return InitResult(lambda0=float(lam0), free=free[: nf.value], fixed_mask=fm,
                      sum_free=float(sj.value))


def simplex_init_lambda(y, r, idx=None, xbar=None, sharpened=False):
    """Algorithm 2, the sequential Gauss-Seidel initializer (simplex.py:114-154).

    Runs the exact recurrence on one device thread (it is inherently serial;
    see par_simplex_init for the chunked form)."""
    if xbar is not None:
        xa = xbar.cpu().numpy() if _is_torch(xbar) else np.asarray(xbar)
        n = int(y.shape[0])
        if xa.shape[0] != n:
            raise DomainError("xbar", None, "xbar must have length n")
        if np.any(xa < 0):
            raise DomainError("xbar", None, "warm-start estimate must be >= 0")
    if idx is not None and len(idx) == 0:
        raise EmptyIndexSet("initializer needs at least one candidate index")
    return _alg2(y, r, idx, xbar, sharpened, workers=1)


def par_simplex_init(y, r, workers=None):
    """Algorithm 2 per contiguous chunk, merged (parallel.py:330-368); one
    device thread per chunk, bit-identical to the reference for the same
    `workers`."""
    from .parallel import resolve_workers

    return _alg2(y, r, None, None, False, workers=resolve_workers(workers))


def _prep(y, keep32=False):
    """(contiguous float64 y -- or float32 with keep32 -- , the caller's dtype, on device)."""
    if _is_torch(y):
        import torch

        if not y.is_cuda:
            y = y.numpy()
        else:
            if y.dtype == torch.float64 and y.is_contiguous():  # the common case: no dispatch
                return y, np.float64, True
            dt = np.float32 if y.dtype == torch.float32 else np.float64
            want = torch.float32 if (keep32 and dt == np.float32) else torch.float64
            return y.to(want).contiguous(), dt, True
    y = np.ascontiguousarray(y)
    if y.dtype not in (np.float32, np.float64):
        y = y.astype(np.float64)
    if keep32 and y.dtype == np.float32:
        return y, y.dtype, False
    return np.ascontiguousarray(y, dtype=np.float64), y.dtype, False


def _project(y, r, opts, lambda0, trace, l1, start="auto", xbar=None, sharpened=None):
    if opts is None:
        opts = SolverOptions()
    # warm start (simplex.py:65-109): Algorithm 2 seeded by xbar's support.
    # A sharpened simplex projection always takes this route: the reference
    # applies the participation test min(y, y + lam) > 0 through
    # simplex_init_lambda (simplex.py:243-245), which changes the answer when
    # lam* > 0.  (For l1, |y| >= 0 and lam* < 0 make the test moot.)
    warm = lambda0 is None and (xbar is not None or (sharpened and (not l1 or start == "alg2")))
    # float32 y: v = y + float(lam) in float (spx_project_f32 / l1_project_f32);
    # the warm routes run the fp64 device Algorithm 2
    yv, dt, dev = _prep(y, keep32=not warm)
    f32 = (str(yv.dtype) == "torch.float32") if dev else yv.dtype == np.float32
    xb = None
    if warm and xbar is not None:
        xb, _, xdev = _prep(xbar)
        if xdev != dev or int(xb.shape[0]) != int(yv.shape[0]):
            raise DomainError("xbar", None, "xbar must match y in length and placement")
        if not bool((xb >= 0).all()):  # simplex.py:139-140 (project_l1 passes xbar as is)
            raise DomainError("xbar", None, "warm-start estimate must be >= 0")
    n = int(yv.shape[0])
    h = N.handle(yv.get_device() if dev else None)
    if dev:
        import torch

        h.use_current_stream()
        x = torch.empty_like(yv)
        yp, xp = yv.data_ptr(), x.data_ptr()
        mem = N.MEM_DEVICE
    else:
        import torch

        h.use_current_stream()
        x = np.empty(n, dtype=np.float32 if f32 else np.float64)
        yp, xp = yv.ctypes.data, x.ctypes.data
        mem = N.MEM_HOST
    o = N.make_options(opts, lambda0=lambda0, trace=trace is not None,
                       compact_ratio=getattr(opts, "compact_ratio", None), start=start, tau=opts.tau(dt))
    res = N.Result()
    if warm:
        xbp = None if xb is None else (xb.data_ptr() if dev else xb.ctypes.data)
        if l1:
            rc = h.lib.l1_project_warm_f64(h.ptr, mem, yp, n, float(r), o, xbp, xp, res)
        else:
            rc = h.lib.spx_project_warm_f64(h.ptr, mem, yp, n, float(r), o, xbp,
                                            1 if sharpened else 0, xp, res)
    elif f32:
        fn = h.lib.l1_project_f32 if l1 else h.lib.spx_project_f32
        rc = fn(h.ptr, mem, yp, n, float(r), o, xp, res)
    else:
        g = N.env_group() if (mem == N.MEM_HOST and trace is None and lambda0 is None) else None
        if g is not None:  # CQK_DEVICES: shard the host vector across the group's GPUs
            fn = g.lib.l1_project_group_f64 if l1 else g.lib.spx_project_group_f64
            with g.lock:
                rc = fn(g.ptr, yp, n, float(r), o, xp, res)
        else:
            fn = h.lib.l1_project_f64 if l1 else h.lib.spx_project_f64
            rc = fn(h.ptr, mem, yp, n, float(r), o, xp, res)
    if trace is not None:
        trace.extend(h.trace(res.trace_len))
    if rc == N.E_DOMAIN:
        what = "l1 radius" if l1 else "simplex level"
        raise DomainError("r", None, f"{what} r must be positive")
    if rc == N.E_CONTRACT:
        raise ContractViolation("zero-size free set in the breakpoint snap")
    if rc != N.SOLVED:
        raise N.NativeError(f"projection failed ({rc}): {N.last_error()}")
    if dt == np.float32 and not f32:
        x = x.float() if dev else x.astype(np.float32)
    return x, res


SPARSE_MIN_N = 4_000_000  # the capture start's size (CQK_SPX_CAPTURE_MIN_N)


def _project_sparse(y, r, opts, l1, start):
    """output="sparse" straight from the device (spx_project_sparse_f64): the
    nonzero x as (index, value) in index order, no dense x.  None when the
    route does not apply (the caller takes the dense one)."""
    if opts is None:
        opts = SolverOptions()
    yv, dt, dev = _prep(y)
    if dt != np.float64:
        return None
    n = int(yv.shape[0])
    if n < SPARSE_MIN_N:
        return None
    cap = min(n // 64 + 1, 1 << 22)
    h = N.handle(yv.get_device() if dev else None)
    h.use_current_stream()
    if dev:
        import torch

        idx = torch.empty(cap, dtype=torch.int64, device=yv.device)
        val = torch.empty(cap, dtype=torch.float64, device=yv.device)
        yp, ip, vp, mem = yv.data_ptr(), idx.data_ptr(), val.data_ptr(), N.MEM_DEVICE
    else:
        idx = np.empty(cap, dtype=np.int64)
        val = np.empty(cap, dtype=np.float64)
        yp, ip, vp, mem = yv.ctypes.data, idx.ctypes.data, val.ctypes.data, N.MEM_HOST
    o = N.make_options(opts, compact_ratio=getattr(opts, "compact_ratio", None), start=start,
                       tau=opts.tau(dt))
    res = N.Result()
    cnt = ctypes.c_int64()
    rc = h.lib.spx_project_sparse_f64(h.ptr, mem, yp, n, float(r), o, 1 if l1 else 0, ip, vp, cap,
                                      ctypes.byref(cnt), res)
    if rc in (N.SPARSE_DENSE, N.SPARSE_OVERFLOW):
        return None
    if rc == N.E_DOMAIN:
        raise DomainError("r", None, ("l1 radius" if l1 else "simplex level") + " r must be positive")
    if rc != N.SOLVED:
        raise N.NativeError(f"sparse projection failed ({rc}): {N.last_error()}")
    k = int(cnt.value)
    return (idx[:k], val[:k]), res


def _sparse(x, dev):
    if dev:
        import torch

        idx = torch.nonzero(x > 0).flatten()
        return idx, x[idx]
    idx = np.flatnonzero(x > 0)
    return idx, x[idx]


def newton_project_simplex(y, r, opts=None, xbar=None, output="dense", sharpened=False,
                           lambda0=None, trace=None, start="auto"):
    """Streamlined Newton projection of y onto the level-r simplex (simplex.py:218-308).

    start (B200 extension, used when lambda0 is None): "auto" (default) =
    the tight start with the first Newton step replaced by a histogram upper
    bound of the root when smaller (fewest passes; the iterate count is this
    route's own); "tight" = min((r - sum y)/n, r - max y) exactly as the
    reference's `lambda0=` route would iterate from it; "formula" =
    (r - sum y)/n (the reference's `lambda0=` formula route); "alg2" = the
    chunked Algorithm-2 initializer (par_simplex_init) with Algorithm 4 on its
    free set.  All routes return the same projection."""
    if not r > 0:
        raise DomainError("r", None, "simplex level r must be positive")
    if output == "sparse" and xbar is None and not sharpened and lambda0 is None and trace is None \
            and start != "alg2":
        got = _project_sparse(y, r, opts, False, start)
        if got is not None:
            sparse, res = got
            return SolveOutcome(status=Status.SOLVED, lam=float(res.lam), x=None,
                                iterations=int(res.iterations), phi_evals=int(res.phi_evals),
                                fixed_count=int(res.fixed_count), sparse=sparse, stats=res.stats())
    x, res = _project(y, r, opts, lambda0, trace, l1=False, start=start, xbar=xbar,
                      sharpened=sharpened)
    dev = _is_torch(x)
    sparse = None
    if output == "sparse":
        sparse = _sparse(x, dev)
        x = None
    return SolveOutcome(status=Status.SOLVED, lam=float(res.lam), x=x,
                        iterations=int(res.iterations), phi_evals=int(res.phi_evals),
                        fixed_count=int(res.fixed_count), sparse=sparse, stats=res.stats())


def project_l1(y, r, opts=None, output="dense", xbar=None, start="auto"):
    """Project y onto the l1 ball of radius r (simplex.py:311-333)."""
    if not r > 0:
        raise DomainError("r", None, "l1 radius r must be positive")
    if output == "sparse" and xbar is None and start != "alg2":
        got = _project_sparse(y, r, opts, True, start)
        if got is not None:
            return got[0]
    try:
        x, res = _project(y, r, opts, None, None, l1=True, start=start, xbar=xbar, sharpened=True)
    except DomainError as e:
        # the reference tests the ball before it looks at xbar
        # (simplex.py:324-327): a point inside is returned even then
        if e.field != "xbar":
            raise
        x, res = _project(y, r, opts, None, None, l1=True, start=start)
        if int(res.iterations) >= 0:
            raise
    if output == "sparse":
        dev = _is_torch(x)
        if dev:
            import torch

            idx = torch.nonzero(x != 0).flatten()
        else:
            idx = np.flatnonzero(x != 0)
        return idx, x[idx]
    return x


def project_l1_outcome(y, r, opts=None, start="auto"):
    """project_l1 with the solver statistics (B200 extension)."""
    x, res = _project(y, r, opts, None, None, l1=True, start=start)
    inside = int(res.iterations) < 0
    return SolveOutcome(status=Status.SOLVED, lam=None if inside else float(res.lam), x=x,
                        iterations=int(res.iterations), phi_evals=int(res.phi_evals),
                        fixed_count=int(res.fixed_count), stats=res.stats())


def project_simplex_rows(Y, r, opts=None, lambda0=None, start="tight", devices=None):
    """Row-wise newton_project_simplex(Y[i], r) for a 2-d array (B200 extension, K8).

    devices (host Y only): a list of CUDA device ordinals; the rows are cut
    into len(devices) contiguous blocks solved concurrently, one per device,
    with no communication (spx_project_batched_multi_f64).  A
    row's result does not depend on the split.

    Returns (X, lam[rows], iterations[rows], stats)."""
    if not r > 0:
        raise DomainError("r", None, "simplex level r must be positive")
    if opts is None:
        opts = SolverOptions()
    dev = _is_torch(Y) and Y.is_cuda
    if devices is None and not dev and N.env_group() is not None:
        devices = list(N.env_group().devices)  # CQK_DEVICES: rows split across the list
    if devices is not None and dev:
        raise ValueError("devices= splits a host array; for CUDA tensors call once per device")
    if dev:
        import torch

        Yv = Y.to(torch.float64).contiguous()
        rows, cols = Yv.shape
        h = N.handle(Yv.device.index)
        h.use_current_stream()
        X = torch.empty_like(Yv)
        lam = torch.empty(rows, dtype=torch.float64, device=Yv.device)
        its = torch.empty(rows, dtype=torch.int32, device=Yv.device)
        ptrs = (Yv.data_ptr(), X.data_ptr(), lam.data_ptr(), its.data_ptr())
        mem = N.MEM_DEVICE
    else:
        Yv = np.ascontiguousarray(Y, dtype=np.float64)
        rows, cols = Yv.shape
        X = np.empty_like(Yv)
        lam = np.empty(rows)
        its = np.empty(rows, np.int32)
        ptrs = (Yv.ctypes.data, X.ctypes.data, lam.ctypes.data, its.ctypes.data)
        mem = N.MEM_HOST
    o = N.make_options(opts, lambda0=lambda0, start=start, tau=opts.tau(np.float64))
    res = N.Result()
    if devices is not None:
        import ctypes

        hs = N.handle_set([int(d) for d in devices])
        arr = (ctypes.c_void_p * len(hs))(*[h.ptr.value for h in hs])
        rc = hs[0].lib.spx_project_batched_multi_f64(arr, len(hs), ptrs[0], rows, cols, float(r), o,
                                                     ptrs[1], ptrs[2], ptrs[3], res)
    else:
        h = N.handle(None) if not dev else h
        h.use_current_stream()
        rc = h.lib.spx_project_batched_f64(h.ptr, mem, ptrs[0], rows, cols, float(r), o, ptrs[1],
                                           ptrs[2], ptrs[3], res)
    if rc != 0:
        raise N.NativeError(f"batched projection failed ({rc}): {N.last_error()}")
    return X, lam, its, res.stats()
