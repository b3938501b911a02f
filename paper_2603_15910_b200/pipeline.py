"""Pipelined host-to-host solves (B200 extension, serving-style throughput).

A stream of CQK instances in host memory is solved `depth` at a time: each
worker thread owns its own library handle (thread-local, with its own staging
buffers and scratch) and its own CUDA stream, so one instance's
host-to-device copy overlaps another's solve and a third's device-to-host
copy of x (the copy engines of the two directions run concurrently).  Every
job is an ordinary solve_cqk call -- same kernels, same results -- and
ctypes releases the GIL for the duration of each call.

    with SolvePipeline(depth=2) as pipe:
        futures = [pipe.submit(inst) for inst in instances]
        outcomes = [f.result() for f in futures]
"""

from concurrent.futures import ThreadPoolExecutor
import threading

from .newton import solve_cqk

__all__ = ["SolvePipeline"]


class SolvePipeline:
    def __init__(self, depth=2, device=None):
        import torch

        self.depth = int(depth)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._tls = threading.local()
        self._pool = ThreadPoolExecutor(max_workers=self.depth, thread_name_prefix="cqk-pipe")
        self.streams = []
        self._lock = threading.Lock()

    def _stream(self):
        import torch

        s = getattr(self._tls, "stream", None)
        if s is None:
            torch.cuda.set_device(self.device)
            s = torch.cuda.Stream(device=self.device)
            self._tls.stream = s
            with self._lock:
                self.streams.append(s)
        return s

    def _run(self, fn, args, kwargs):
        import torch

        s = self._stream()
        with torch.cuda.stream(s):
            return fn(*args, **kwargs)

    def submit(self, inst, opts=None, xbar=None, check=True, fn=solve_cqk):
        """Queue one solve; returns a concurrent.futures.Future of its SolveOutcome."""
        return self._pool.submit(self._run, fn, (inst,), {"opts": opts, "xbar": xbar, "check": check})

    def close(self):
        self._pool.shutdown(wait=True)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
