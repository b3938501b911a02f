"""Multi-GPU sharded solves: one process (and one cqk handle) per GPU.

Replaces the reference's chunked fork-join drivers (parallel.py:174-327 with
contiguous chunks, parallel.py:82-85, and the fixed-order _tree_sum,
parallel.py:62-72) at node scale: rank q owns the contiguous shard
[n*q/W, n*(q+1)/W) of every array and runs the same persistent kernel as the
single-GPU solve on it.  The cross-GPU step is fused into that kernel: once per
Newton epoch one warp of each rank stores its partial-sum vector into every
peer's mailbox over NVLink (CUDA IPC mapped device memory; lane k stores value
k to all peers, one system-scope fence, lane q raises peer q's flag), and every
CTA reduces the W vectors in rank order, so all ranks take the identical
decision with no collective library call and no host round trip.  torch.distributed is used
once, at set-up, to exchange the 64-byte IPC handles.
"""

import ctypes

import numpy as np

from . import _native as N
from .core import DomainError
from .newton import SolverOptions, _outcome

__all__ = ["shard_bounds", "Communicator", "ShardedCQK", "ShardedProjection",
           "sharded_projection", "local_group"]

_VARIANTS = {"solve": N.VARIANT_SOLVE, "jacobi": N.VARIANT_JACOBI, "par": N.VARIANT_PAR}


def shard_bounds(n, world, rank):
    """Contiguous equal shard of rank `rank` (the reference's _chunk_ranges split)."""
    return n * rank // world, n * (rank + 1) // world


def allgather_bytes(payload, group=None):
    """All ranks' byte strings, in rank order (torch.distributed plumbing)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(payload), group=group)
    return out


class Communicator:
    """Mailbox set-up for a handle.  `peers`: same-process handles (virtual
    ranks, e.g. several handles on one GPU); otherwise IPC handles are
    exchanged over torch.distributed (`group`)."""

    def __init__(self, handle, rank, world, group=None, peers=None):
        self.handle, self.rank, self.world = handle, int(rank), int(world)
        lib = handle.lib
        size = lib.cqk_comm_ipc_handle_size()
        buf = ctypes.create_string_buffer(size)
        rc = lib.cqk_comm_create(handle.ptr, self.rank, self.world,
                                 None if peers is not None else buf)
        if rc != 0:
            raise N.NativeError(f"cqk_comm_create failed ({rc}): {N.last_error()}")
        self._peers = peers
        if peers is None and self.world > 1:
            blobs = allgather_bytes(buf.raw, group)
            joined = b"".join(blobs)
            rc = lib.cqk_comm_connect(handle.ptr, joined)
            if rc != 0:
                raise N.NativeError(f"cqk_comm_connect failed ({rc}): {N.last_error()}")

    def connect_local(self):
        arr = (ctypes.c_void_p * self.world)(*[h.ptr.value for h in self._peers])
        rc = self.handle.lib.cqk_comm_connect_local(self.handle.ptr, arr, self.world)
        if rc != 0:
            raise N.NativeError(f"cqk_comm_connect_local failed ({rc}): {N.last_error()}")


def local_group(devices, grid_limit=None):
    """W same-process ranks (handles) wired to each other -- for one-node
    set-ups that run all ranks in one process, and for testing the exchange
    on a single GPU with `grid_limit` CTAs per rank."""
    handles = [N.Handle(dv) for dv in devices]
    if grid_limit:
        for h in handles:
            h.lib.cqk_set_grid_limit(h.ptr, int(grid_limit))
    comms = [Communicator(h, q, len(handles), peers=handles) for q, h in enumerate(handles)]
    for c in comms:
        c.connect_local()
    return comms


def _ptrs(tensors):
    return [None if t is None else t.data_ptr() for t in tensors]


class ShardedCQK:
    """This rank's shard of a CQK instance, resident on its GPU.

    arrays: CUDA tensors (d, a, b, l, u) of the shard; r, n_total, offset of
    the global instance.  `solve` is collective: every rank calls it with the
    same options and gets the same status / lambda / counters, and x for its
    own shard."""

    launches_per_solve = 1

    def __init__(self, arrays, r, n_total, offset, comm=None, group=None):
        import torch
        import torch.distributed as dist

        self.arrays = [a.to(torch.float64).contiguous() for a in arrays]
        self.n_local = int(self.arrays[0].numel())
        self.r, self.n_total, self.offset = float(r), int(n_total), int(offset)
        self.device = self.arrays[0].device.index
        if comm is None:
            h = N.handle(self.device)
            comm = Communicator(h, dist.get_rank(group), dist.get_world_size(group), group=group)
        self.comm = comm
        self.handle = comm.handle
        # no allocation may happen inside a collective solve: a cudaMalloc can
        # synchronise the device while the peers' kernels wait on this rank
        rc = self.handle.lib.cqk_reserve(self.handle.ptr, self.n_local)
        if rc != 0:
            raise N.NativeError(f"cqk_reserve failed ({rc}): {N.last_error()}")
        self.x = torch.empty(self.n_local, dtype=torch.float64, device=f"cuda:{self.device}")
        torch.cuda.synchronize(self.device)

    def solve(self, opts=None, variant="solve", check=True, xbar=None, want_x=True):
        """Collective solve; x is this rank's shard, written into a buffer
        owned by this object (valid until the next solve)."""
        import torch

        if opts is None:
            opts = SolverOptions()
        h = self.handle
        h.use_current_stream()
        x = self.x if want_x else None
        o = N.make_options(opts, variant=_VARIANTS[variant], check=check,
                           compact_ratio=getattr(opts, "compact_ratio", None),
                           fixing=False if variant == "jacobi" else None, tau=opts.tau(np.float64))
        res = N.Result()
        xb = None if xbar is None else xbar.to(torch.float64).contiguous()
        rc = h.lib.cqk_solve_sharded_f64(h.ptr, N.MEM_DEVICE, *_ptrs(self.arrays), self.n_local,
                                         self.offset, self.n_total, self.r, o,
                                         None if xb is None else xb.data_ptr(),
                                         None if x is None else x.data_ptr(), res)

        class _I:  # dtype carrier for _outcome
            dtype = np.dtype(np.float64)

        return _outcome(_I, res, rc, x, "sharded solve_cqk")

    def solve_host(self, host_arrays, x_out=None, opts=None, variant="solve", check=True):
        """Collective solve of this rank's shard given in HOST memory (numpy,
        ideally page-locked): the library copies it to the device, solves and
        writes x back into x_out (a host array of n_local, allocated if None)."""
        import torch

        if opts is None:
            opts = SolverOptions()
        h = self.handle
        if not getattr(self, "_host_reserved", False):
            rc = h.lib.cqk_reserve_host(h.ptr, self.n_local)
            if rc != 0:
                raise N.NativeError(f"cqk_reserve_host failed ({rc}): {N.last_error()}")
            self._host_reserved = True
        h.use_current_stream()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in host_arrays]
        if x_out is None:
            x_out = torch.empty(self.n_local, dtype=torch.float64, pin_memory=True).numpy()
        o = N.make_options(opts, variant=_VARIANTS[variant], check=check,
                           compact_ratio=getattr(opts, "compact_ratio", None),
                           fixing=False if variant == "jacobi" else None, tau=opts.tau(np.float64))
        res = N.Result()
        rc = h.lib.cqk_solve_sharded_f64(h.ptr, N.MEM_HOST, *[a.ctypes.data for a in arrs],
                                         self.n_local, self.offset, self.n_total, self.r, o, None,
                                         x_out.ctypes.data, res)

        class _I:
            dtype = np.dtype(np.float64)

        return _outcome(_I, res, rc, x_out, "sharded solve_cqk")


class ShardedProjection:
    """This rank's shard of y for collective simplex (l1=False) / l1-ball
    projections (newton_project_simplex / project_l1 over n_total)."""

    launches_per_solve = 1

    def __init__(self, comm, y_local, n_total):
        import torch

        self.comm, self.handle = comm, comm.handle
        self.y = y_local.to(torch.float64).contiguous()
        self.n_total = int(n_total)
        rc = self.handle.lib.cqk_reserve(self.handle.ptr, int(self.y.numel()))
        if rc != 0:
            raise N.NativeError(f"cqk_reserve failed ({rc}): {N.last_error()}")
        self.x = torch.empty_like(self.y)
        torch.cuda.synchronize(self.y.device)

    def solve(self, r, l1=False, opts=None, start="tight"):
        import torch

        from .newton import SolveOutcome, Status

        if not r > 0:
            raise DomainError("r", None, "radius / level r must be positive")
        if opts is None:
            opts = SolverOptions()
        h = self.handle
        h.use_current_stream()
        o = N.make_options(opts, compact_ratio=getattr(opts, "compact_ratio", None), start=start,
                           tau=opts.tau(np.float64))
        res = N.Result()
        fn = h.lib.l1_project_sharded_f64 if l1 else h.lib.spx_project_sharded_f64
        rc = fn(h.ptr, N.MEM_DEVICE, self.y.data_ptr(), int(self.y.numel()), self.n_total,
                float(r), o, self.x.data_ptr(), res)
        if rc != 0:
            raise N.NativeError(f"sharded projection failed ({rc}): {N.last_error()}")
        inside = int(res.iterations) < 0
        return SolveOutcome(status=Status.SOLVED, lam=None if inside else float(res.lam),
                            x=self.x, iterations=int(res.iterations),
                            phi_evals=int(res.phi_evals), fixed_count=int(res.fixed_count),
                            stats=res.stats())

    def solve_host(self, y_host, r, l1=False, opts=None, start="tight", x_out=None):
        """Collective projection of this rank's shard given in HOST memory
        (numpy, ideally page-locked): H2D, the persistent kernel, D2H of x."""
        if not r > 0:
            raise DomainError("r", None, "radius / level r must be positive")
        if opts is None:
            opts = SolverOptions()
        h = self.handle
        if not getattr(self, "_host_reserved", False):
            rc = h.lib.cqk_reserve_host(h.ptr, int(self.y.numel()))
            if rc != 0:
                raise N.NativeError(f"cqk_reserve_host failed ({rc}): {N.last_error()}")
            self._host_reserved = True
        h.use_current_stream()
        yv = np.ascontiguousarray(y_host, dtype=np.float64)
        if x_out is None:
            x_out = np.empty_like(yv)
        o = N.make_options(opts, compact_ratio=getattr(opts, "compact_ratio", None), start=start,
                           tau=opts.tau(np.float64))
        res = N.Result()
        fn = h.lib.l1_project_sharded_f64 if l1 else h.lib.spx_project_sharded_f64
        rc = fn(h.ptr, N.MEM_HOST, yv.ctypes.data, int(yv.size), self.n_total, float(r), o,
                x_out.ctypes.data, res)
        if rc != 0:
            raise N.NativeError(f"sharded projection failed ({rc}): {N.last_error()}")
        return x_out, res.stats()


def sharded_projection(comm, y_local, n_total, r, l1=False, opts=None):
    """One-shot collective projection (allocates; prefer ShardedProjection)."""
    return ShardedProjection(comm, y_local, n_total).solve(r, l1=l1, opts=opts)
