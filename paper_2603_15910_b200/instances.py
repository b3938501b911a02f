"""Seeded benchmark instance generators (drop-in for cqksolve.instances).

Backed by lib/libcqk_instances.so (csrc/instances.c): Xoshiro256++ with the
reference's seeding and draw order (instances.py:43-86, rng.py:29-106),
parallelised over host cores with GF(2) skip-ahead.  Arrays are bit-identical
to the reference's; the CQK level r is formed with pairwise dot products
rather than the reference's BLAS ddot, so it can differ in the last bits.
"""

import ctypes

import numpy as np

from . import _native as N
from .core import CqkInstance

__all__ = ["CQK_FAMILIES", "SIMPLEX_FAMILIES", "FamilyMismatch", "gen_cqk", "gen_simplex_y",
           "gen_blobs", "gen_sparse_ls", "gen_cqk_device", "gen_simplex_y_device", "Xoshiro256pp"]

CQK_FAMILIES = ("cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated")
SIMPLEX_FAMILIES = ("simplex-u01", "simplex-n01", "simplex-n0m3")


class FamilyMismatch(ValueError):
    """Generator asked for a family it does not produce."""


def gen_cqk_arrays(family, n, seed, out=None):
    """(d, a, b, l, u, r) as float64 arrays; `out` may supply 5 preallocated arrays."""
    if family not in CQK_FAMILIES:
        raise FamilyMismatch(f"not a CQK family: {family!r}")
    arrs = out if out is not None else [np.empty(n) for _ in range(5)]
    r = ctypes.c_double()
    rc = N.gen_library().cqk_gen_cqk(CQK_FAMILIES.index(family), int(n), int(seed) & (2**64 - 1),
                                     *[a.ctypes.data for a in arrs], ctypes.byref(r))
    if rc != 0:
        raise ValueError(f"gen_cqk failed ({rc})")
    return (*arrs, float(r.value))


def gen_cqk_shard(family, n, seed, lo, hi):
    """Elements [lo, hi) of gen_cqk(family, n, seed) without generating the rest
    (GF(2) skip-ahead): (d, a, b, l, u, bl, bu) with this shard's pairwise
    b.l / b.u sums; combine the shards' sums with `cqk_r`."""
    if family not in CQK_FAMILIES:
        raise FamilyMismatch(f"not a CQK family: {family!r}")
    m = int(hi) - int(lo)
    arrs = [np.empty(m) for _ in range(5)]
    bl, bu = ctypes.c_double(), ctypes.c_double()
    rc = N.gen_library().cqk_gen_cqk_range(CQK_FAMILIES.index(family), int(n),
                                           int(seed) & (2**64 - 1), int(lo), int(hi),
                                           *[a.ctypes.data for a in arrs], ctypes.byref(bl),
                                           ctypes.byref(bu))
    if rc != 0:
        raise ValueError(f"gen_cqk_shard failed ({rc})")
    return (*arrs, float(bl.value), float(bu.value))


def cqk_r(family, n, seed, bl, bu):
    """r = b.l + U (b.u - b.l) with the stream's final draw (instances.py:64-66)."""
    return float(N.gen_library().cqk_gen_cqk_r(CQK_FAMILIES.index(family), int(n),
                                               int(seed) & (2**64 - 1), float(bl), float(bu)))


def gen_cqk(family, n, seed, dtype=np.float64):
    """One random CQK instance of the given family (instances.py:43-70)."""
    d, a, b, l, u, r = gen_cqk_arrays(family, n, seed)
    return CqkInstance(d=d.astype(dtype), a=a.astype(dtype), b=b.astype(dtype),
                       l=l.astype(dtype), u=u.astype(dtype), r=r)


def gen_simplex_y(family, n, seed, dtype=np.float64):
    """One random point for the simplex benchmarks (instances.py:73-86)."""
    if family not in SIMPLEX_FAMILIES:
        raise FamilyMismatch(f"not a simplex family: {family!r}")
    y = np.empty(int(n))
    rc = N.gen_library().cqk_gen_simplex_y(SIMPLEX_FAMILIES.index(family), int(n),
                                           int(seed) & (2**64 - 1), y.ctypes.data)
    if rc != 0:
        raise ValueError(f"gen_simplex_y failed ({rc})")
    return y.astype(dtype)


class Xoshiro256pp:
    """Seeded xoshiro256++ stream (rng.py:82-106), random access by draw offset."""

    def __init__(self, seed):
        self.seed = int(seed) & (2**64 - 1)
        self.pos = 0

    def uniform01(self, size):
        out = np.empty(int(size))
        N.gen_library().cqk_gen_uniform01(self.seed, self.pos, out.size, out.ctypes.data)
        self.pos += out.size
        return out

    def uniform(self, lo, hi, size):
        return lo + self.uniform01(size) * (hi - lo)

    def normal(self, size, std=1.0):
        out = np.empty(int(size))
        N.gen_library().cqk_gen_normal(self.seed, self.pos, out.size, out.ctypes.data)
        self.pos += 2 * out.size
        if std != 1.0:
            out *= std
        return out

    def integers(self, upper, size):
        u = self.uniform01(size)
        return np.minimum((u * upper).astype(np.int64), upper - 1)


def gen_blobs(n, dim, separation, seed):
    """Two Gaussian blobs labelled +1 (even i) / -1 (odd i) for the SVM-dual
    SPG demo (instances.py:89-101): n*dim normals in point-major order, then
    the class mean +-separation/2 added to coordinate 0."""
    g = Xoshiro256pp(seed)
    pts = g.normal(int(n) * int(dim)).reshape(int(n), int(dim))
    labels = np.where(np.arange(int(n)) % 2 == 0, 1.0, -1.0)
    pts[:, 0] += 0.5 * separation * labels
    return pts, labels


def gen_sparse_ls(m, n, density, sparsity_k, seed):
    """Sparse least squares (A CSR, b = A x_true, x_true) for the basis-pursuit
    SPG demo (instances.py:103-131).  Stream order: m*n uniforms (entry kept
    below `density`), one normal per kept entry in row-major order, support
    indices drawn one at a time (a repeat is redrawn), then sparsity_k
    normals for the support values."""
    import scipy.sparse as sp

    from .core import DomainError

    if not 0 < density <= 1:
        raise DomainError("density", None, "density must be in (0, 1]")
    if sparsity_k > n:
        raise DomainError("sparsity_k", None, "sparsity_k must be <= n")
    g = Xoshiro256pp(seed)
    keep = g.uniform01(int(m) * int(n)) < density
    rows, cols = np.nonzero(keep.reshape(int(m), int(n)))
    A = sp.csr_matrix((g.normal(rows.shape[0]), (rows, cols)), shape=(int(m), int(n)))
    support, seen = [], set()
    while len(support) < sparsity_k:
        c = int(g.integers(int(n), 1)[0])
        if c not in seen:
            seen.add(c)
            support.append(c)
    x_true = np.zeros(int(n))
    if sparsity_k:
        x_true[np.array(support)] = g.normal(int(sparsity_k))
    return A, A @ x_true, x_true


def gen_cqk_device(family, n, seed, device=None):
    """gen_cqk straight into CUDA memory: bit-identical arrays (per-thread
    GF(2) jumps of the Xoshiro256++ stream), r from device b.l / b.u sums.
    Returns a CqkInstance of CUDA tensors."""
    import torch

    if family not in CQK_FAMILIES:
        raise FamilyMismatch(f"not a CQK family: {family!r}")
    h = N.handle(device)
    h.use_current_stream()
    arrs = [torch.empty(int(n), dtype=torch.float64, device=f"cuda:{h.device}") for _ in range(5)]
    r = ctypes.c_double()
    rc = h.lib.cqk_gen_cqk_device(h.ptr, CQK_FAMILIES.index(family), int(n),
                                  int(seed) & (2**64 - 1), *[t.data_ptr() for t in arrs],
                                  ctypes.byref(r))
    if rc != 0:
        raise N.NativeError(f"device generator failed ({rc}): {N.last_error()}")
    return CqkInstance(*arrs, r=float(r.value))


def gen_cqk_shard_device(family, n, seed, lo, hi, device=None):
    """Elements [lo, hi) of gen_cqk(family, n, seed) generated in CUDA memory:
    ([d, a, b, l, u] tensors, bl, bu) -- combine the shards' b.l / b.u with
    cqk_r to get the instance's r."""
    import torch

    if family not in CQK_FAMILIES:
        raise FamilyMismatch(f"not a CQK family: {family!r}")
    h = N.handle(device)
    h.use_current_stream()
    arrs = [torch.empty(int(hi) - int(lo), dtype=torch.float64, device=f"cuda:{h.device}")
            for _ in range(5)]
    bl, bu = ctypes.c_double(), ctypes.c_double()
    rc = h.lib.cqk_gen_cqk_device_range(h.ptr, CQK_FAMILIES.index(family), int(n),
                                        int(seed) & (2**64 - 1), int(lo), int(hi),
                                        *[t.data_ptr() for t in arrs], ctypes.byref(bl),
                                        ctypes.byref(bu))
    if rc != 0:
        raise N.NativeError(f"device generator failed ({rc}): {N.last_error()}")
    return arrs, float(bl.value), float(bu.value)


def gen_simplex_y_device(family, n, seed, device=None):
    """gen_simplex_y into CUDA memory: simplex-u01 is generated on the device
    (bit-identical); the normal families use the host generator (their
    Box-Muller log/cos must be glibc's to stay bit-identical) and one copy."""
    import torch

    if family not in SIMPLEX_FAMILIES:
        raise FamilyMismatch(f"not a simplex family: {family!r}")
    h = N.handle(device)
    if family != "simplex-u01":
        return torch.from_numpy(gen_simplex_y(family, n, seed)).to(f"cuda:{h.device}")
    h.use_current_stream()
    y = torch.empty(int(n), dtype=torch.float64, device=f"cuda:{h.device}")
    rc = h.lib.cqk_gen_simplex_u01_device(h.ptr, int(n), int(seed) & (2**64 - 1), y.data_ptr())
    if rc != 0:
        raise N.NativeError(f"device generator failed ({rc}): {N.last_error()}")
    return y
