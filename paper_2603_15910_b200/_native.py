"""ctypes binding of the in-tree native libraries.

``libcqk_b200.so`` is the only compute path: there is no CPU fallback, and
every entry point raises ``NativeUnavailable`` when the library (or a CUDA
device) is missing.  ``libcqk_instances.so`` holds the host-side instance
generators.
"""

import ctypes
import math
import os
import threading

import numpy as np

from . import build as _build

LIB_PATH = _build.CUDA_LIB
GEN_PATH = _build.GEN_LIB

SOLVED, INFEASIBLE = 0, 1
E_DOMAIN, E_MAXITER, E_CONTRACT, E_CUDA, E_ARG, E_EMPTY, E_TIMEOUT = -1, -2, -3, -4, -5, -6, -7
MEM_HOST, MEM_DEVICE = 0, 1
VARIANT_SOLVE, VARIANT_JACOBI, VARIANT_PAR = 0, 1, 2
FIELDS = ("d", "a", "b", "l", "u", "r", "bounds", "y", "xbar")


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing -- there is no fallback."""


class NativeError(RuntimeError):
    """A CUDA / argument error reported by the native library."""


class Options(ctypes.Structure):
    _fields_ = [
        ("variable_fixing", ctypes.c_int32),
        ("max_iterations", ctypes.c_int32),
        ("tolerance_scale", ctypes.c_double),
        ("variant", ctypes.c_int32),
        ("check", ctypes.c_int32),
        ("lambda0", ctypes.c_double),
        ("compact_ratio", ctypes.c_double),
        ("record_trace", ctypes.c_int32),
        ("simplex_start", ctypes.c_int32),
    ]


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
        ("elems_read", ctypes.c_int64),
        ("elems_written", ctypes.c_int64),
        ("bytes_model", ctypes.c_int64),
        ("device_ms", ctypes.c_double),
        ("launches", ctypes.c_int32),
        ("trace_len", ctypes.c_int32),
    ]

    def stats(self):
        return {
            "elems_read": int(self.elems_read),
            "elems_written": int(self.elems_written),
            "bytes_model": int(self.bytes_model),
            "device_ms": float(self.device_ms),
            "launches": int(self.launches),
            "lam0": float(self.lam0),
            "bracket": (float(self.bracket_lo), float(self.bracket_hi)),
        }


# Every symbol declared in include/cqk_b200.h (checked by the CPU tests).
EXPORTS = (
    "cqk_abi_version", "cqk_last_error", "cqk_create", "cqk_destroy", "cqk_set_stream",
    "cqk_device_info", "cqk_get_trace", "cqk_get_timeline", "cqk_validate_f64", "cqk_initial_multiplier_f64",
    "cqk_phi_f64", "cqk_eval_x_f64", "cqk_nearest_breakpoint_f64", "cqk_solve_f64",
    "spx_project_f64", "l1_project_f64", "spx_project_warm_f64", "l1_project_warm_f64",
    "spx_project_batched_f64", "cqk_selftest_division",
    "cqk_comm_ipc_handle_size", "cqk_comm_create", "cqk_comm_connect", "cqk_comm_connect_local",
    "cqk_set_grid_limit", "cqk_set_engine", "cqk_set_fused", "cqk_set_fused_guess", "cqk_set_switches", "cqk_reserve", "cqk_reserve_host", "cqk_solve_sharded_f64", "spx_project_sharded_f64",
    "l1_project_sharded_f64", "spx_init_alg2_f64", "cqk_gen_cqk_device",
    "cqk_gen_cqk_device_range", "cqk_gen_simplex_u01_device", "spx_project_batched_multi_f64",
    "cqk_read_peak_f64", "cqk_group_create", "cqk_group_destroy", "cqk_group_size",
    "cqk_solve_group_f64", "spx_project_group_f64", "l1_project_group_f64",
    "cqk_solve_f32", "spx_project_f32", "l1_project_f32", "spx_project_sparse_f64",
)
SPARSE_DENSE, SPARSE_OVERFLOW = 2, 3

_lib = None
_gen = None
_lock = threading.Lock()
_tls = threading.local()

_P = ctypes.c_void_p
_D = ctypes.c_double
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_RES = ctypes.POINTER(Result)
_OPT = ctypes.POINTER(Options)


def _declare(L):
    L.cqk_abi_version.restype = ctypes.c_int
    L.cqk_last_error.restype = ctypes.c_char_p
    L.cqk_create.argtypes = [ctypes.POINTER(_P), ctypes.c_int]
    L.cqk_destroy.argtypes = [_P]
    L.cqk_set_stream.argtypes = [_P, _P]
    L.cqk_device_info.argtypes = [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                  ctypes.POINTER(_I32)]
    L.cqk_get_trace.argtypes = [_P, _P, _I32]
    L.cqk_get_timeline.argtypes = [_P, _P, _I32]
    arr5 = [_P] * 5
    L.cqk_validate_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _D, _RES]
    L.cqk_initial_multiplier_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _D, _P,
                                             ctypes.POINTER(_D)]
    L.cqk_phi_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _P, _I64, _D, _P, _P, _P]
    L.cqk_eval_x_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _P, _I64, _D, _P]
    L.cqk_nearest_breakpoint_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _P, _I64, _D,
                                             ctypes.c_int, ctypes.POINTER(_D),
                                             ctypes.POINTER(_I32)]
    L.cqk_solve_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _D, _OPT, _P, _P, _RES]
    L.spx_project_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, _P, _RES]
    L.l1_project_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, _P, _RES]
    L.spx_project_warm_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, _P, ctypes.c_int,
                                       _P, _RES]
    L.l1_project_warm_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, _P, _P, _RES]
    L.cqk_selftest_division.argtypes = [_P, ctypes.c_uint64, _I64, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_uint64), _P]
    L.cqk_comm_ipc_handle_size.restype = ctypes.c_int
    L.cqk_comm_create.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P]
    L.cqk_comm_connect.argtypes = [_P, _P]
    L.cqk_comm_connect_local.argtypes = [_P, _P, ctypes.c_int]
    L.cqk_set_grid_limit.argtypes = [_P, ctypes.c_int]
    L.cqk_set_engine.argtypes = [_P, ctypes.c_int]
    L.cqk_set_fused.argtypes = [_P, _I64, _D]
    L.cqk_set_fused_guess.argtypes = [_P, ctypes.c_int]
    L.cqk_set_switches.argtypes = [_P, ctypes.c_int]
    L.cqk_reserve_host.argtypes = [_P, _I64]
    L.cqk_reserve.argtypes = [_P, _I64]
    L.cqk_solve_sharded_f64.argtypes = [_P, ctypes.c_int, *arr5, _I64, _I64, _I64, _D, _OPT, _P,
                                        _P, _RES]
    L.spx_project_sharded_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _I64, _D, _OPT, _P, _RES]
    L.l1_project_sharded_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _I64, _D, _OPT, _P, _RES]
    L.spx_init_alg2_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _P, _I64, _I64, _P,
                                    ctypes.c_int, ctypes.POINTER(_D), ctypes.POINTER(_I64), _P,
                                    _P, ctypes.POINTER(_D), ctypes.POINTER(_I64)]
    L.cqk_gen_cqk_device.argtypes = [_P, ctypes.c_int, _I64, ctypes.c_uint64, _P, _P, _P, _P,
                                     _P, ctypes.POINTER(_D)]
    L.cqk_gen_simplex_u01_device.argtypes = [_P, _I64, ctypes.c_uint64, _P]
    L.cqk_gen_cqk_device_range.argtypes = [_P, ctypes.c_int, _I64, ctypes.c_uint64, _I64, _I64,
                                           _P, _P, _P, _P, _P, ctypes.POINTER(_D),
                                           ctypes.POINTER(_D)]
    L.spx_project_batched_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _I64, _D, _OPT, _P, _P,
                                          _P, _RES]
    L.spx_project_batched_multi_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _I64, _D, _OPT, _P,
                                                _P, _P, _RES]
    L.spx_project_sparse_f64.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, ctypes.c_int, _P, _P,
                                         _I64, ctypes.POINTER(_I64), _RES]
    L.cqk_solve_f32.argtypes = [_P, ctypes.c_int, *arr5, _I64, _D, _OPT, _P, _P, _RES]
    L.spx_project_f32.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, _P, _RES]
    L.l1_project_f32.argtypes = [_P, ctypes.c_int, _P, _I64, _D, _OPT, _P, _RES]
    L.cqk_group_create.argtypes = [ctypes.POINTER(_P), _P, ctypes.c_int]
    L.cqk_group_destroy.argtypes = [_P]
    L.cqk_group_size.argtypes = [_P]
    L.cqk_solve_group_f64.argtypes = [_P, *arr5, _I64, _D, _OPT, _P, _P, _RES]
    L.spx_project_group_f64.argtypes = [_P, _P, _I64, _D, _OPT, _P, _RES]
    L.l1_project_group_f64.argtypes = [_P, _P, _I64, _D, _OPT, _P, _RES]
    L.cqk_read_peak_f64.argtypes = [_P, _P, ctypes.c_int, _I64, ctypes.c_int, ctypes.POINTER(_D),
                                    ctypes.POINTER(_D)]


def load_library(path=None):
    """Load (not build) libcqk_b200.so; raises NativeUnavailable if absent."""
    global _lib
    with _lock:
        if _lib is None:
            p = path or os.environ.get("CQK_LIB") or LIB_PATH
            if not os.path.exists(p):
                raise NativeUnavailable(
                    f"{p} is missing: run `python -m paper_2603_15910_b200.build` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(p)
            _declare(L)
            _lib = L
    return _lib


def gen_library():
    global _gen
    with _lock:
        if _gen is None:
            if not os.path.exists(GEN_PATH):
                _build.build_instances()
            G = ctypes.CDLL(GEN_PATH)
            G.cqk_gen_uniform01.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _I64, _P]
            G.cqk_gen_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _I64, _P]
            G.cqk_gen_cqk.argtypes = [ctypes.c_int, _I64, ctypes.c_uint64, _P, _P, _P, _P, _P,
                                      ctypes.POINTER(_D)]
            G.cqk_gen_simplex_y.argtypes = [ctypes.c_int, _I64, ctypes.c_uint64, _P]
            G.cqk_gen_cqk_range.argtypes = [ctypes.c_int, _I64, ctypes.c_uint64, _I64, _I64,
                                            _P, _P, _P, _P, _P, ctypes.POINTER(_D),
                                            ctypes.POINTER(_D)]
            G.cqk_gen_cqk_r.argtypes = [ctypes.c_int, _I64, ctypes.c_uint64, _D, _D]
            G.cqk_gen_cqk_r.restype = _D
            _gen = G
    return _gen


def last_error():
    return (load_library().cqk_last_error() or b"").decode()


class Handle:
    """One cqk_handle (device-bound; not re-entrant)."""

    def __init__(self, device=0):
        import torch  # plumbing only: device discovery and streams

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible (the solver has no CPU fallback)")
        L = load_library()
        h = _P()
        rc = L.cqk_create(ctypes.byref(h), int(device))
        if rc != 0:
            raise NativeError(f"cqk_create failed ({rc}): {last_error()}")
        self.ptr = h
        self.device = int(device)
        self.lib = L

    def set_stream(self, stream_ptr):
        """Bind to a cudaStream_t; 0 (torch's default stream) maps to
        cudaStreamLegacy so work stays ordered with the caller's stream."""
        self.lib.cqk_set_stream(self.ptr, _P(stream_ptr if stream_ptr else 1))
        self._stream = stream_ptr

    def set_fused(self, min_n=4_000_000, half_width=2e-3, guess=1):
        """Fused start of the CQK solve from `min_n` elements per rank, with
        the direction guess mode `guess` (cqk_b200.h)."""
        if self.lib.cqk_set_fused(self.ptr, int(min_n), float(half_width)) != 0:
            raise NativeError(last_error())
        if self.lib.cqk_set_fused_guess(self.ptr, int(guess)) != 0:
            raise NativeError(last_error())

    def set_switches(self, master_step=False, static_final=False, tail=True, capture=True,
                     capture_fail=False):
        """A/B switches of the persistent kernels (cqk_set_switches)."""
        flags = ((1 if master_step else 0) | (2 if static_final else 0) | (0 if tail else 4)
                 | (0 if capture else 8) | (16 if capture_fail else 0))
        if self.lib.cqk_set_switches(self.ptr, flags) != 0:
            raise NativeError(last_error())

    def use_current_stream(self):
        """Bind to torch's current stream on this handle's device (the C call
        only when it changed)."""
        s = _current_raw_stream(self.device)
        if s != getattr(self, "_stream", None):
            self.set_stream(s)

    def info(self):
        sm, ctas, thr = _I32(), _I32(), _I32()
        self.lib.cqk_device_info(self.ptr, ctypes.byref(sm), ctypes.byref(ctas), ctypes.byref(thr))
        return {"sm_count": sm.value, "ctas": ctas.value, "threads": thr.value}

    def trace(self, rows):
        out = np.zeros((max(rows, 1), 4))
        got = self.lib.cqk_get_trace(self.ptr, out.ctypes.data, int(rows))
        return [tuple(float(v) for v in row) for row in out[: max(got, 0)]]

    def timeline(self, rows=64):
        """Per-pass device timeline of the last persistent solve (see cqk_b200.h)."""
        out = np.zeros((rows, 20), dtype=np.int64)
        got = self.lib.cqk_get_timeline(self.ptr, out.ctypes.data, int(rows))
        return out[: max(got, 0)]

    def read_peak(self, tensors, reps=5):
        """Read-only streaming ceiling (GB/s, ms) over equal-length fp64 CUDA
        tensors on this handle's device (cqk_read_peak_f64)."""
        n = int(tensors[0].numel())
        arr = (_P * len(tensors))(*[t.data_ptr() for t in tensors])
        gbs, ms = _D(), _D()
        self.use_current_stream()
        rc = self.lib.cqk_read_peak_f64(self.ptr, arr, len(tensors), n, int(reps), ctypes.byref(gbs),
                                        ctypes.byref(ms))
        if rc != 0:
            raise NativeError(f"cqk_read_peak_f64 failed ({rc}): {last_error()}")
        return gbs.value, ms.value

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                self.lib.cqk_destroy(self.ptr)
        except Exception:
            pass


def _current_raw_stream(device):
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(device))
    return torch.cuda.current_stream(device).cuda_stream


def handle(device=None):
    """Thread-local handle for `device` (default: torch's current device)."""
    import torch

    if device is None:
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible (the solver has no CPU fallback)")
        device = torch.cuda.current_device()
    cache = getattr(_tls, "handles", None)
    if cache is None:
        cache = _tls.handles = {}
    h = cache.get(device)
    if h is None:
        h = cache[device] = Handle(device)
    return h


def handle_set(devices):
    """One distinct handle per list entry (a device may appear several
    times), cached per thread -- for calls that drive several handles at once
    (spx_project_batched_multi_f64)."""
    key = tuple(devices)
    cache = getattr(_tls, "sets", None)
    if cache is None:
        cache = _tls.sets = {}
    hs = cache.get(key)
    if hs is None:
        hs = cache[key] = [Handle(d) for d in devices]
    return hs


class Group:
    """A same-process device group (cqk_group, include/cqk_b200.h): one rank
    per listed device, solves over host arrays sharded across them."""

    def __init__(self, devices):
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible (the solver has no CPU fallback)")
        self.lib = load_library()
        self.devices = tuple(int(d) for d in devices)
        arr = (ctypes.c_int * len(self.devices))(*self.devices)
        g = _P()
        rc = self.lib.cqk_group_create(ctypes.byref(g), arr, len(self.devices))
        if rc != 0:
            raise NativeError(f"cqk_group_create failed ({rc}): {last_error()}")
        self.ptr = g
        self.lock = threading.Lock()  # a group is not re-entrant

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                self.lib.cqk_group_destroy(self.ptr)
        except Exception:
            pass


_groups = {}
_glock = threading.Lock()


def parse_devices(spec):
    """CQK_DEVICES syntax: comma-separated CUDA ordinals ("0,1,2,3"; a device
    may repeat to host several ranks)."""
    out = [int(t) for t in str(spec).replace(" ", "").split(",") if t != ""]
    if any(d < 0 for d in out):
        raise ValueError(f"bad device list {spec!r}")
    return out


def env_group():
    """The process-wide group of CQK_DEVICES when it lists >= 2 entries, else
    None (the GPU analogue of CQK_WORKERS, parallel.py:52-59)."""
    spec = os.environ.get("CQK_DEVICES")
    if not spec:
        return None
    devs = tuple(parse_devices(spec))
    if len(devs) < 2:
        return None
    with _glock:
        g = _groups.get(devs)
        if g is None:
            g = _groups[devs] = Group(devs)
    return g


_OPTS_CACHE = {}
_START = {"formula": 0, "tight": 1, "alg2": 2, "auto": 4}


def make_options(opts=None, variant=VARIANT_SOLVE, check=True, lambda0=None,
                 compact_ratio=None, trace=False, fixing=None, start="auto", tau=None):
    """The C options struct (tau: the tolerance the solve uses).  Structs are
    cached by value and shared: callers must not mutate the result."""
    fix = getattr(opts, "variable_fixing", True) if fixing is None else fixing
    max_it = int(getattr(opts, "max_iterations", 100))
    ts = tau if tau is not None else getattr(opts, "tolerance_scale", None)
    key = (bool(fix), max_it, ts, variant, bool(check), lambda0, compact_ratio, bool(trace), start)
    o = _OPTS_CACHE.get(key)
    if o is not None:
        return o
    o = Options()
    o.variable_fixing = 1 if fix else 0
    o.max_iterations = max_it
    o.tolerance_scale = float(ts) if ts is not None else math.nan
    o.variant = variant
    o.check = 1 if check else 0
    o.lambda0 = math.nan if lambda0 is None else float(lambda0)
    o.compact_ratio = math.nan if compact_ratio is None else float(compact_ratio)
    o.record_trace = 1 if trace else 0
    o.simplex_start = _START[start]
    if len(_OPTS_CACHE) > 1024:
        _OPTS_CACHE.clear()
    _OPTS_CACHE[key] = o
    return o
