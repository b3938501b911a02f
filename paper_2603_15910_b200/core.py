"""Problem data, the dual map x(lambda) and the dual residual phi(lambda).

Drop-in for cqksolve.core (/root/reference/pkg/src/cqksolve/core.py).  The
types keep the reference's fields and coercions; the data-parallel work
(validate, eval_phi, eval_x, initial_multiplier, breakpoints) runs in the
sm_100a library through the C-ABI.  Instance arrays may be numpy arrays
(host; staged through HBM per call) or CUDA torch tensors (device-resident,
zero-copy).
"""

from dataclasses import dataclass

import numpy as np

from . import _native as N

__all__ = [
    "DomainError",
    "CqkInstance",
    "SimplexInstance",
    "PhiEval",
    "Breakpoints",
    "validate",
    "eval_x",
    "eval_phi",
    "initial_multiplier",
    "breakpoints",
    "simplex_as_cqk",
]


class DomainError(ValueError):
    """Problem data violates an invariant (bad sign, l > u, NaN, ...).  core.py:30-36"""

    def __init__(self, field, index, message):
        self.field = field
        self.index = index
        super().__init__(message)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _coerce(v, dt):
    if _is_torch(v):
        import torch

        tdt = torch.float32 if dt == np.float32 else torch.float64
        return v.to(tdt).contiguous()
    return np.ascontiguousarray(v, dtype=dt)


def _dtype_of(v):
    if _is_torch(v):
        import torch

        return np.dtype(np.float32) if v.dtype == torch.float32 else np.dtype(np.float64)
    dt = np.asarray(v).dtype
    return dt if dt in (np.float32, np.float64) else np.dtype(np.float64)


@dataclass
class CqkInstance:
    """Data (d, a, b, l, u, r) of one CQK instance (core.py:39-76).

    Arrays share a common length n and floating dtype; -inf in l and +inf in
    u are allowed.  Treated as immutable after construction.
    """

    d: object
    a: object
    b: object
    l: object
    u: object
    r: float

    def __post_init__(self):
        dt = _dtype_of(self.d)
        self.d = _coerce(self.d, dt)
        self.a = _coerce(self.a, dt)
        self.b = _coerce(self.b, dt)
        self.l = _coerce(self.l, dt)
        self.u = _coerce(self.u, dt)
        self.r = dt.type(self.r)

    @property
    def n(self):
        return int(self.d.shape[0])

    @property
    def dtype(self):
        return _dtype_of(self.d)

    @property
    def eps(self):
        return float(np.finfo(self.dtype).eps)


@dataclass
class SimplexInstance:
    """A point y to project onto {x >= 0, sum x = r} (core.py:79-100)."""

    y: object
    r: float

    def __post_init__(self):
        if _is_torch(self.y):
            self.y = _coerce(self.y, _dtype_of(self.y))
            import torch

            finite = bool(torch.isfinite(self.y).all())
            ny = self.y.dim()
            size = self.y.shape[0] if ny == 1 else 0
        else:
            self.y = np.ascontiguousarray(self.y)
            if self.y.dtype not in (np.float32, np.float64):
                self.y = self.y.astype(np.float64)
            finite = None
            ny = self.y.ndim
            size = self.y.shape[0] if ny == 1 else 0
        if ny != 1 or size < 1:
            raise DomainError("y", None, "y must be a nonempty 1-d array")
        if finite is None:
            finite = bool(np.all(np.isfinite(self.y)))
        if not finite:
            yy = self.y.cpu().numpy() if _is_torch(self.y) else self.y
            idx = int(np.flatnonzero(~np.isfinite(yy))[0])
            raise DomainError("y", idx, f"y[{idx}] is not finite")
        if not self.r > 0:
            raise DomainError("r", None, f"simplex level r must be positive, got {self.r}")

    @property
    def n(self):
        return int(self.y.shape[0])


@dataclass
class PhiEval:
    """phi(lam) together with both lateral derivatives at lam (core.py:103-109)."""

    value: float
    dminus: float
    dplus: float


@dataclass
class Breakpoints:
    """Finite slope-change locations of phi with their variable indices."""

    lower: np.ndarray
    lower_idx: np.ndarray
    upper: np.ndarray
    upper_idx: np.ndarray


# ------------------------------------------------------------- marshalling
class Marshal:
    """Pointers for the C-ABI: numpy -> host mode (fp64 staging), CUDA torch
    tensors -> device mode (zero-copy).  float64 by default; f32=True keeps
    float32 instances float32 for the *_f32 entry points (the reference
    computes float32 instances in float32, core.py:55-64, 195-200)."""

    def __init__(self, *arrays, f32=False):
        """f32: keep float32 arrays float32 (the *_f32 entry points)."""
        self.torch = any(_is_torch(a) for a in arrays if a is not None)
        self.keep = []
        self.ptrs = []
        self.f32 = f32
        if self.torch:
            import torch

            dev = None
            for a in arrays:
                if a is None:
                    self.ptrs.append(None)
                    continue
                if not _is_torch(a) or not a.is_cuda:
                    raise ValueError("mixing CUDA tensors with host arrays is not supported")
                want = torch.float32 if f32 else torch.float64
                t = a if a.dtype == want and a.is_contiguous() else a.to(want).contiguous()
                dev = t.device if dev is None else dev
                self.keep.append(t)
                self.ptrs.append(t.data_ptr())
            self.device = dev.index if dev is not None else 0
            self.mem = N.MEM_DEVICE
        else:
            for a in arrays:
                if a is None:
                    self.ptrs.append(None)
                    continue
                v = np.ascontiguousarray(a, dtype=np.float32 if f32 else np.float64)
                self.keep.append(v)
                self.ptrs.append(v.ctypes.data)
            self.device = None
            self.mem = N.MEM_HOST

    def handle(self):
        """Handle bound to torch's current stream on the target device, so
        callers can order and time solves with ordinary torch events."""
        import torch

        h = N.handle(self.device)
        h.use_current_stream()
        return h

    def empty(self, n):
        import torch

        tdt = torch.float32 if self.f32 else torch.float64
        if self.torch:
            t = torch.empty(n, dtype=tdt, device=f"cuda:{self.device}")
            return t, t.data_ptr()
        # host results land in page-locked memory (torch's caching host
        # allocator), so the device-to-host copy of x runs at full DMA rate
        v = torch.empty(n, dtype=tdt, pin_memory=True).numpy()
        return v, v.ctypes.data

    def index(self, idx, n):
        if idx is None:
            return None, None, n
        if self.torch:
            import torch

            t = torch.as_tensor(idx, device=f"cuda:{self.device}").to(torch.int64).contiguous()
            return t, t.data_ptr(), int(t.numel())
        v = np.ascontiguousarray(idx, dtype=np.int64)
        return v, v.ctypes.data, int(v.size)


def _cast_out(x, dtype):
    if x is None:
        return None
    if dtype == np.float32:
        return x.float() if _is_torch(x) else x.astype(np.float32)
    return x


def _raise_native(h, rc, what):
    raise N.NativeError(f"{what} failed ({rc}): {N.last_error()}")


def raise_domain(res):
    field = N.FIELDS[res.domain_field] if 0 <= res.domain_field < len(N.FIELDS) else "?"
    idx = int(res.domain_index) if res.domain_index >= 0 else None
    if field == "bounds":
        msg = f"l[{idx}] > u[{idx}]"
    elif idx is None:
        msg = f"{field} violates its domain"
    else:
        msg = f"{field}[{idx}] violates its domain"
    raise DomainError(field, idx, msg)


# ------------------------------------------------------------- functions
def validate(inst):
    """Raise DomainError on the first violated invariant (core.py:126-165), on device."""
    if inst.n < 1:
        raise DomainError("d", None, "instance must have at least one variable")
    for name in ("d", "a", "b", "l", "u"):
        arr = getattr(inst, name)
        if len(arr.shape) != 1 or arr.shape[0] != inst.n:
            raise DomainError(name, None, f"{name} must be 1-d of length {inst.n}")
    m = Marshal(inst.d, inst.a, inst.b, inst.l, inst.u)
    h = m.handle()
    res = N.Result()
    rc = h.lib.cqk_validate_f64(h.ptr, m.mem, *m.ptrs, inst.n, float(inst.r), res)
    if rc == N.E_DOMAIN:
        raise_domain(res)
    if rc != 0:
        _raise_native(h, rc, "validate")


def eval_x(inst, lam, idx=None):
    """The primal minimizer x(lam) clipped to [l, u] (core.py:168-179); idx selects components."""
    m = Marshal(inst.d, inst.a, inst.b, inst.l, inst.u)
    ix, ixp, cnt = m.index(idx, inst.n)
    h = m.handle()
    x, xp = m.empty(cnt)
    lamv = float(inst.dtype.type(lam))
    rc = h.lib.cqk_eval_x_f64(h.ptr, m.mem, *m.ptrs, inst.n, ixp, cnt, lamv, xp)
    if rc != 0:
        _raise_native(h, rc, "eval_x")
    return _cast_out(x, inst.dtype)


def phi_scan(inst, lam, idx=None, masks=False):
    """core.py:182-212 _phi_scan on device -> (value, dminus, dplus, abs_bx[, at_lower, at_upper])."""
    m = Marshal(inst.d, inst.a, inst.b, inst.l, inst.u)
    ix, ixp, cnt = m.index(idx, inst.n)
    h = m.handle()
    out = np.zeros(4)
    lo = hi = None
    lop = hip = None
    if masks:
        if m.torch:
            import torch

            lo = torch.empty(cnt, dtype=torch.uint8, device=f"cuda:{m.device}")
            hi = torch.empty(cnt, dtype=torch.uint8, device=f"cuda:{m.device}")
            lop, hip = lo.data_ptr(), hi.data_ptr()
        else:
            lo = np.empty(cnt, np.uint8)
            hi = np.empty(cnt, np.uint8)
            lop, hip = lo.ctypes.data, hi.ctypes.data
    lamv = float(inst.dtype.type(lam))
    rc = h.lib.cqk_phi_f64(h.ptr, m.mem, *m.ptrs, inst.n, ixp, cnt, lamv, out.ctypes.data, lop, hip)
    if rc != 0:
        _raise_native(h, rc, "eval_phi")
    vals = (float(out[0]), float(out[1]), float(out[2]), float(out[3]))
    if masks:
        return vals + (lo.bool(), hi.bool()) if m.torch else vals + (lo.astype(bool), hi.astype(bool))
    return vals


def eval_phi(inst, lam, idx=None):
    """phi(lam) = b'x(lam) and both lateral derivatives (core.py:215-225)."""
    value, dminus, dplus, _ = phi_scan(inst, lam, idx)
    return PhiEval(value=value, dminus=dminus, dplus=dplus)


def breakpoints(inst):
    """All finite breakpoints (d*bound - a)/b with their variable indices (core.py:228-234).

    Host-side utility (not on the Newton hot path)."""
    d, a, b, l, u = (np.asarray(v.cpu().numpy() if _is_torch(v) else v)
                     for v in (inst.d, inst.a, inst.b, inst.l, inst.u))
    fin_l = np.flatnonzero(np.isfinite(l))
    fin_u = np.flatnonzero(np.isfinite(u))
    lower = (d[fin_l] * l[fin_l] - a[fin_l]) / b[fin_l]
    upper = (d[fin_u] * u[fin_u] - a[fin_u]) / b[fin_u]
    return Breakpoints(lower=lower, lower_idx=fin_l, upper=upper, upper_idx=fin_u)


def initial_multiplier(inst, xbar=None):
    """(r - sum b*a/d) / sum b^2/d over all indices or the interior of xbar (core.py:237-257)."""
    if xbar is not None:
        shape = tuple(xbar.shape) if hasattr(xbar, "shape") else np.asarray(xbar).shape
        if shape != (inst.n,):
            raise DomainError("xbar", None, "xbar must have length n")
    m = Marshal(inst.d, inst.a, inst.b, inst.l, inst.u, xbar)
    h = m.handle()
    out = ctypes_double()
    rc = h.lib.cqk_initial_multiplier_f64(h.ptr, m.mem, *m.ptrs[:5], inst.n, float(inst.r),
                                          m.ptrs[5], out)
    if rc != 0:
        _raise_native(h, rc, "initial_multiplier")
    return float(out.value)


def ctypes_double():
    import ctypes

    return ctypes.c_double()


def simplex_as_cqk(y, r):
    """Embed a simplex projection as a CQK instance (d=b=1, l=0, u=inf); core.py:260-274."""
    if _is_torch(y):
        import torch

        y = y.contiguous()
        if y.dtype not in (torch.float32, torch.float64):
            y = y.to(torch.float64)
        one = torch.ones_like(y)
        return CqkInstance(d=one, a=y, b=one.clone(), l=torch.zeros_like(y),
                           u=torch.full_like(y, float("inf")), r=r)
    y = np.ascontiguousarray(y)
    if y.dtype not in (np.float32, np.float64):
        y = y.astype(np.float64)
    n = y.shape[0]
    one = np.ones(n, dtype=y.dtype)
    return CqkInstance(d=one, a=y, b=one.copy(), l=np.zeros(n, dtype=y.dtype),
                       u=np.full(n, np.inf, dtype=y.dtype), r=r)
