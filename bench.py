#!/usr/bin/env python
"""Headline benchmark: CQK n=1e8 fp64 solve (BASELINE.json configs[2], C3).

One "step" = one complete solve_cqk (variable fixing, the reference's default
driver) of the cqk-weakly-correlated n = 1e8 instance (seed 1, generated
bit-identically to the reference's Xoshiro256++ stream), inputs resident in
HBM.  4 GB of inputs > 126 MB L2, so no flush is needed between steps.

  value   elements/s = n * K / (device time of K steps), max over ranks
  e2e     the same metric through the public API with pinned HOST buffers
          (H2D of d,a,b,l,u + solve + D2H of x inside the timed region)
  roofline achieved = algorithmic bytes per launch of the persistent solve
          kernel (SURVEY 8(d) byte model, counted by the kernel) / its
          CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline the C oracle (restatement of the reference) on this host

`--impl reference` times the reference's CPU algorithm (the oracle port of
par_solve_cqk, all host threads) on a bounded sample of the same workload.
N > 1 (torchrun): n is sharded over the ranks (strong scaling); every
Newton iteration exchanges the partial-sum vector between ranks.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FAMILY = "cqk-weakly-correlated"
N_FULL = 10**8
SEED = 1
METRIC = "elements/sec and % HBM roofline, CQK n=1e8 fp64 solve at 1/2/4/8 B200 vs CPU"
UNIT = "elements/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 3 + k and r[3 + k].lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * (max(smax) if smax else 1)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CQK_BENCH_DEVICE / CQK_BENCH_BACKEND=gloo: run the N>1 code path with all
    # ranks on one GPU (a smoke test of the sharded protocol, not a number)
    if os.environ.get("CQK_BENCH_DEVICE") is not None:
        local = int(os.environ["CQK_BENCH_DEVICE"])
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        backend = os.environ.get("CQK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gen_shard(n_total, world, rank):
    """This rank's contiguous shard of the instance (generated directly with
    GF(2) skip-ahead) and the global r from the shards' b.l / b.u sums."""
    import paper_2603_15910_b200 as P

    if world == 1:
        d, a, b, l, u, r = P.instances.gen_cqk_arrays(FAMILY, n_total, SEED)
        return [d, a, b, l, u], r, 0, n_total
    from paper_2603_15910_b200.distributed import allgather_bytes, shard_bounds

    lo, hi = shard_bounds(n_total, world, rank)
    # the shard is generated straight into this rank's HBM (bit-identical stream)
    dev, bl, bu = P.instances.gen_cqk_shard_device(FAMILY, n_total, SEED, lo, hi)
    parts = [np.frombuffer(x, dtype=np.float64) for x in
             allgather_bytes(np.array([bl, bu]).tobytes())]
    sbl = sbu = 0.0
    for pbl, pbu in parts:  # rank order: identical on every rank
        sbl += pbl
        sbu += pbu
    r = P.instances.cqk_r(FAMILY, n_total, SEED, sbl, sbu)
    return dev, r, lo, hi


def cpu_baseline_sample(arrs, r, cores):
    """C oracle restatement of solve_cqk (1 thread) on the first 1e7 elements
    of the instance (a bounded sample; r rescaled to keep it feasible)."""
    import oracle

    oracle.build()
    m = min(10**7, arrs[0].size)
    d, a, b, l, u = (v[:m] for v in arrs)
    bl, bu = float(b @ l), float(b @ u)
    rs = bl + 0.5 * (bu - bl)
    t0 = time.perf_counter()
    out = oracle.solve_cqk(d, a, b, l, u, rs, fixing=True, want_x=True)
    dt = time.perf_counter() - t0
    assert out["status"] == 0
    return {"value": m / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle solve_cqk (C restatement of newton.solve_cqk, fixing, 1 thread) on the "
                      f"first {m} elements of the {FAMILY} instance, r at mid-range; {dt:.2f} s"}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on the host cores (oracle port)."""
    if rank != 0:
        return
    import oracle
    import paper_2603_15910_b200 as P

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    m = args.ref_sample
    d, a, b, l, u, r = P.instances.gen_cqk_arrays(FAMILY, m, SEED)
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = oracle.par_solve_cqk(d, a, b, l, u, r, workers=cores, fixing=True)
        dt = time.perf_counter() - t0
        assert out["status"] == 0
        if k >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = m * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference Xoshiro256++ stream, bit-identical inputs)",
        "config": {"workload": f"C3 {FAMILY} solve (par_solve_cqk, fixing), bounded sample n={m}",
                   "family": FAMILY, "n": m, "seed": SEED},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"oracle par_solve_cqk (C/OpenMP restatement of parallel.py:174-327) "
                                   f"with {cores} threads on n={m} of {FAMILY}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--size", dest="n", type=int, default=N_FULL)
    ap.add_argument("--variant", default="solve", choices=["solve", "jacobi"])
    ap.add_argument("--ref-sample", type=int, default=10**7)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch

    import paper_2603_15910_b200 as P

    torch.cuda.set_device(local)
    arrs, r, lo, hi = gen_shard(args.n, world, rank)
    n_local = hi - lo
    stream = torch.cuda.Stream()
    if world == 1:
        with torch.cuda.stream(stream):
            dev = [torch.from_numpy(v).cuda() for v in arrs]
        stream.synchronize()
    else:
        dev = arrs  # already resident (generated on the device)
    if world > 1:
        from paper_2603_15910_b200 import distributed as D

        solver = D.ShardedCQK(dev, r, n_total=args.n, offset=lo)
        solve = lambda: solver.solve(variant=args.variant)  # noqa: E731
    else:
        inst = P.CqkInstance(*dev, r=r)
        if args.variant == "solve":
            solve = lambda: P.solve_cqk(inst)  # noqa: E731
        else:
            solve = lambda: P.jacobi_solve(inst)  # noqa: E731

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            out = solve()
        assert out.status is P.Status.SOLVED
        stream.synchronize()
        barrier(world)
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.15)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        kern_ms, bytes_model, evals, iters = [], [], [], []
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            out = solve()
            kern_ms.append(out.stats["device_ms"])
            bytes_model.append(out.stats["bytes_model"])
            evals.append(out.phi_evals)
            iters.append(out.iterations)
        ev1.record(stream)
        torch.cuda.synchronize()
        clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, world)
    value = args.n * args.steps / (ms / 1e3)

    hbm, peak_src = peaks()
    kms = statistics.mean(kern_ms)
    bpl = statistics.mean(bytes_model)
    achieved = bpl / (kms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_solve_kernel.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e through the public API with pinned host buffers (H2D + solve + D2H
    # inside every step).  Measured twice: sequential solve_cqk calls, and the
    # public SolvePipeline (depth 2: one step's H2D overlaps the previous
    # step's solve and D2H -- each step still moves all its bytes).
    e2e = None
    if world > 1 and args.e2e_steps > 0:
        # every rank: its shard's H2D from pinned host memory + the collective
        # solve + D2H of its x, device-timed, max over ranks
        host = [t.cpu().pin_memory().numpy() for t in dev]
        xh = torch.empty(n_local, dtype=torch.float64, pin_memory=True).numpy()
        with torch.cuda.stream(stream):
            for _ in range(2):
                assert solver.solve_host(host, xh).status is P.Status.SOLVED
            torch.cuda.synchronize()
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.e2e_steps):
                assert solver.solve_host(host, xh).status is P.Status.SOLVED
            e1.record(stream)
            torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, world)
        e2e = {"value": args.n / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 5 * 8 * args.n, "d2h_bytes_per_step": 8 * args.n,
               "ms_per_step": ems, "api": "ShardedCQK.solve_host (each rank its shard)"}
        del host
    if world == 1 and args.e2e_steps > 0:
        from paper_2603_15910_b200.pipeline import SolvePipeline

        pinned = [torch.from_numpy(v).pin_memory() for v in arrs]
        host = [t.numpy() for t in pinned]
        inst_h = P.CqkInstance(*host, r=r)

        def seq_ms():
            with torch.cuda.stream(stream):
                # warm-up: the caching host allocator ends up holding the two
                # pinned x blocks a steady-state caller cycles through
                for _ in range(3):
                    out = P.solve_cqk(inst_h)
                    del out
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.e2e_steps):
                    out = P.solve_cqk(inst_h)  # H2D of d,a,b,l,u + solve + D2H of x
                    assert out.status is P.Status.SOLVED
                    del out
                e1.record(stream)
                torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.e2e_steps

        def pipe_ms(depth):
            import collections

            def run(steps, pipe):
                # a bounded window, results consumed (and their pinned x
                # released) in order -- a steady-state serving loop
                q = collections.deque()
                for _ in range(steps):
                    q.append(pipe.submit(inst_h))
                    if len(q) > depth:
                        assert q.popleft().result().status is P.Status.SOLVED
                while q:
                    assert q.popleft().result().status is P.Status.SOLVED

            with SolvePipeline(depth=depth) as pipe:
                run(3 * depth, pipe)  # warm-up: handles, staging, pinned blocks
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                run(args.e2e_steps, pipe)
                for s_ in pipe.streams:
                    stream.wait_stream(s_)
                e1.record(stream)
                torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.e2e_steps

        ms_seq = seq_ms()
        ms_pipe = pipe_ms(2)
        e2e = {"value": args.n / (ms_pipe / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 5 * 8 * args.n, "d2h_bytes_per_step": 8 * args.n,
               "ms_per_step": ms_pipe, "api": "SolvePipeline(depth=2).submit -> solve_cqk",
               "sequential": {"value": args.n / (ms_seq / 1e3), "ms_per_step": ms_seq,
                              "api": "solve_cqk, one call after another"}}
        del pinned, host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample(arrs, r, 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference Xoshiro256++ stream, bit-identical inputs)",
            "config": {
                "workload": f"C3 {FAMILY} n={args.n} solve_cqk "
                            f"({'variable fixing' if args.variant == 'solve' else 'jacobi'})",
                "family": FAMILY, "n": args.n, "seed": SEED,
                "parallelism": f"shard n over {world} GPU(s)" if world > 1 else "single GPU",
                "l2": "inputs 4 GB > 126 MB L2; no flush needed",
                "phi_evals": statistics.mode(evals), "iterations": statistics.mode(iters),
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "cqk_tma_kernel<true> (persistent TMA-pipelined solve, 1 launch/solve)",
                         "bytes_per_launch": bpl, "kernel_ms": kms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": args.steps * (1 if world == 1 else solver.launches_per_solve),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
