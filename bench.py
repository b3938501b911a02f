#!/usr/bin/env python
"""Headline benchmark: CQK n=1e8 fp64 solve (BASELINE.json configs[2], C3).

One "step" = one complete solve_cqk (variable fixing, the reference's default
driver) of one n = 1e8 instance; the steps rotate through six resident
instances -- cqk-weakly-correlated and cqk-correlated, seeds 1-3 (BASELINE.md
section 2: three C3 instances per family) -- generated bit-identically to the
reference's Xoshiro256++ stream.  4 GB per instance > 126 MB L2: no flush is
needed between steps.

  value        elements/s = n * K / (device time of K steps), max over ranks
  e2e          the same metric through the public API with pinned HOST buffers
               (H2D of d,a,b,l,u + solve + D2H of x inside the timed region)
  roofline     algorithmic bytes per launch of the persistent solve kernel
               (SURVEY 8(d) byte model, counted by the kernel) / its CUDA-event
               duration, against MEASURED_PEAKS.json hbm_gbs (the copy peak);
               `peak_read` is the read-only streaming ceiling measured in this
               run by the library's bulk-copy stream kernel
  cpu_baseline the C oracle's solve_cqk (1 thread) on the SAME first instance
               (same arrays, same r), its lambda checked against the GPU's

`--impl reference` times the reference's CPU algorithm on the box's host cores
(the oracle's C/OpenMP par_solve_cqk, all threads) on the SAME instances: they
are rebuilt by the oracle's own generator (oracle/cqk_gen.c), so that arm loads
no product library.  Both arms print an identical `config`.

N > 1: run under torchrun (or pass --gpus N: the script relaunches itself with
torch.distributed.run).  C3 shards n over the ranks (every Newton iteration
exchanges the partial-sum vector inside the kernel over NVLink); `--config c4`
(l1 ball, n = 1e9) shards y the same way; `--config c5` (65536 x 4096 rows)
splits the rows with no communication.
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "elements/sec and % HBM roofline, CQK n=1e8 fp64 solve at 1/2/4/8 B200 vs CPU"
UNIT = "elements/s"
WEAK, CORR = "cqk-weakly-correlated", "cqk-correlated"
DATA = "synthetic (reference Xoshiro256++ stream, bit-identical inputs)"
NCU_SOLVE = os.path.join(ROOT, "profiles", "r02_ncu_solve.json")

CONFIGS = {
    "c3": {"kind": "cqk", "n": 10**8,
           "instances": [(WEAK, 1), (WEAK, 2), (WEAK, 3), (CORR, 1), (CORR, 2), (CORR, 3)],
           "metric": METRIC},
    "c4": {"kind": "l1", "n": 10**9, "family": "simplex-n01", "seed": 1, "r": 1.0,
           "metric": "elements/sec and % HBM roofline, l1-ball projection n=1e9 fp64 (C4)"},
    "c5": {"kind": "rows", "rows": 65536, "cols": 4096, "family": "simplex-n01", "seed": 1, "r": 1.0,
           "metric": "elements/sec and % HBM roofline, batched simplex 65536x4096 fp64 (C5)"},
}


def bench_config(name, cfg, world, n_override=None):
    """The workload description -- identical in both arms at the same N."""
    par = f"{world} GPU(s)"
    if cfg["kind"] == "cqk":
        n = n_override or cfg["n"]
        return {"workload": f"C3 solve_cqk (variable fixing) n={n}, one of "
                            f"{len(cfg['instances'])} instances per step in rotation",
                "n": n, "instances": [f"{f}:seed{s}" for f, s in cfg["instances"]],
                "r": "b.l + U (b.u - b.l), b.l / b.u numpy-pairwise sums (identical in both arms)",
                "parallelism": f"shard n over {par}" if world > 1 else "single GPU",
                "l2": "inputs 4 GB per instance > 126 MB L2; no flush needed"}
    if cfg["kind"] == "l1":
        n = n_override or cfg["n"]
        return {"workload": f"C4 project_l1(y, r=1) n={n}, y = gen_simplex_y(simplex-n01, seed 1)",
                "n": n, "instances": [f"{cfg['family']}:seed{cfg['seed']}"], "r": cfg["r"],
                "parallelism": f"shard y over {par}" if world > 1 else "single GPU",
                "l2": "8 GB input > 126 MB L2; no flush needed"}
    rows = n_override or cfg["rows"]
    return {"workload": f"C5 row-wise newton_project_simplex(Y[i], 1), {rows} x {cfg['cols']}",
            "rows": rows, "cols": cfg["cols"], "n": rows * cfg["cols"],
            "instances": [f"{cfg['family']}:seed{cfg['seed']}"], "r": cfg["r"],
            "parallelism": f"rows split over {par}, no communication" if world > 1 else "single GPU",
            "l2": "2 GB input > 126 MB L2; no flush needed"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
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


# ------------------------------------------------------------------ plumbing
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args):
    """--gpus N without a torchrun environment: relaunch as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # CQK_BENCH_DEVICE: every rank on that one GPU (a protocol smoke test of the
    # sharded path on a one-GPU box, not a number)
    if os.environ.get("CQK_BENCH_DEVICE") is not None:
        local = int(os.environ["CQK_BENCH_DEVICE"])
    if world > 1 and args.impl != "reference":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        # NCCL refuses two ranks on one device: the one-GPU smoke test uses gloo
        shared = os.environ.get("CQK_BENCH_DEVICE") is not None
        backend = os.environ.get("CQK_BENCH_BACKEND", "gloo" if shared else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def reduce_max(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def broadcast_obj(obj, world):
    if world == 1:
        return obj
    import torch.distributed as dist

    box = [obj]
    dist.broadcast_object_list(box, src=0)
    return box[0]


# ------------------------------------------------------------------ reference arm
def run_reference(args, name, cfg, world, rank):
    """The reference's CPU algorithm on this host's cores, on the same inputs
    (oracle generator: no product library is loaded by this arm)."""
    if rank != 0:
        return
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    config = bench_config(name, cfg, world, args.n)
    budget = args.ref_budget
    times, per_inst, warm = [], [], 0
    t_start = time.perf_counter()
    if cfg["kind"] == "cqk":
        n = config["n"]
        insts = cfg["instances"]
        alg = f"oracle par_solve_cqk (C/OpenMP restatement of parallel.py:174-327), {cores} threads"
        for i, (fam, seed) in enumerate(insts):
            mine = [k for k in range(args.steps) if k % len(insts) == i]
            if not mine:
                continue
            d, a, b, l, u, r = oracle.gen_cqk(fam, n, seed)
            run = lambda: oracle.par_solve_cqk(d, a, b, l, u, r, workers=cores, fixing=True,  # noqa: E731
                                               want_x=True)
            for _ in range(max(1, -(-args.warmup // len(insts)))):
                assert run()["status"] == 0
                warm += 1
            lam = None
            for _ in mine:
                t0 = time.perf_counter()
                out = run()
                times.append(time.perf_counter() - t0)
                assert out["status"] == 0
                lam = out["lam"]
            per_inst.append({"instance": f"{fam}:seed{seed}", "lam": lam,
                             "iterations": out["iterations"], "phi_evals": out["phi_evals"]})
            del d, a, b, l, u
    elif cfg["kind"] == "l1":
        n = config["n"]
        alg = "oracle project_l1 (C restatement of simplex.py:311-333; the reference's l1 path is sequential), 1 thread"
        cores_used = 1
        y = oracle.gen_simplex_y(cfg["family"], n, cfg["seed"])
        assert oracle.project_l1(y, cfg["r"])["status"] == 0
        warm = 1
        for _ in range(args.steps):
            t0 = time.perf_counter()
            out = oracle.project_l1(y, cfg["r"])
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > budget:
                break
        per_inst.append({"instance": config["instances"][0], "lam": out["lam"],
                         "iterations": out["iterations"]})
        cores = cores_used
    else:
        rows, cols = config["rows"], config["cols"]
        n = rows * cols
        alg = f"oracle newton_project_simplex per row (simplex.py:218-308), OpenMP over rows, {cores} threads"
        Y = oracle.gen_simplex_y(cfg["family"], n, cfg["seed"]).reshape(rows, cols)
        assert oracle.project_simplex_rows(Y, cfg["r"], threads=cores)[3] == 0
        warm = 1
        for _ in range(args.steps):
            t0 = time.perf_counter()
            _, lam, its, bad = oracle.project_simplex_rows(Y, cfg["r"], threads=cores)
            times.append(time.perf_counter() - t0)
            assert bad == 0
            if time.perf_counter() - t_start > budget:
                break
        per_inst.append({"instance": config["instances"][0], "lam_row0": float(lam[0]),
                         "iterations_mean": float(its.mean())})
    tot = sum(times)
    value = n * len(times) / tot
    line = {
        "impl": "reference", "metric": cfg["metric"], "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "warmup": warm, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": DATA, "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{alg}; the full workload, {len(times)} timed steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "results": per_inst,
        "host": {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm helpers
class Timed:
    """K steps bracketed by a barrier + synchronize, CUDA events on `stream`,
    nvidia-smi clocks sampled throughout; per-step library stats collected."""

    def __init__(self, world, local, stream):
        self.world, self.local, self.stream = world, local, stream

    def run(self, steps, step):
        import torch

        torch.cuda.synchronize()
        barrier(self.world)
        sampler = ClockSampler(self.local)
        sampler.start()
        time.sleep(0.15)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        outs = []
        torch.cuda.synchronize()
        ev0.record(self.stream)
        for k in range(steps):
            outs.append(step(k))
        ev1.record(self.stream)
        torch.cuda.synchronize()
        clocks = sampler.stop()
        ms = reduce_max(ev0.elapsed_time(ev1), self.world)
        return ms, outs, clocks


def ncu_traffic():
    """DRAM bytes per launch of the committed ncu --set full capture."""
    try:
        with open(NCU_SOLVE) as f:
            rec = json.load(f)
        return rec.get("dram_bytes_per_launch"), rec.get("algorithmic_bytes_per_launch")
    except Exception:
        return None, None


def roofline(outs, world, read_peak, kernel, traffic=None):
    hbm, src = peaks()
    kms = statistics.mean(o["device_ms"] for o in outs)
    bpl = statistics.mean(o["bytes_model"] for o in outs)
    achieved = bpl / (kms / 1e3) / 1e9
    rl = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
          "traffic": traffic, "peak_source": src, "kernel": kernel,
          "bytes_per_launch": bpl, "kernel_ms": kms, "per": "rank 0's kernel" if world > 1 else "GPU"}
    if read_peak:
        rl["peak_read"] = read_peak
        rl["frac_read"] = achieved / read_peak
        rl["peak_read_source"] = ("measured in this run: cqk_read_peak_f64 (bulk-copy read-only "
                                  "stream of the 5 resident arrays, best of 5)")
    return rl


def cqk_instances(cfg, n, world, rank, local):
    """Resident instances (this rank's shard of each) + rank 0's host copy of
    the first one.  r is the instance's r over all n (rank 0 generates the full
    instance on the host and broadcasts r), identical at every N."""
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200.distributed import shard_bounds

    lo, hi = shard_bounds(n, world, rank)
    dev, host0, rs = [], None, []
    for i, (fam, seed) in enumerate(cfg["instances"]):
        r = None
        if rank == 0:
            arrs = P.instances.gen_cqk_arrays(fam, n, seed)
            r = arrs[5]
            if i == 0:
                host0 = arrs
        r = broadcast_obj(r, world)
        rs.append(r)
        if world == 1:
            d = [torch.from_numpy(v).cuda() for v in arrs[:5]]
        else:
            d, _, _ = P.instances.gen_cqk_shard_device(fam, n, seed, lo, hi, device=local)
        dev.append(d)
        if rank == 0 and i > 0:
            del arrs
    torch.cuda.synchronize()
    return dev, rs, host0, (lo, hi)


def cpu_baseline_cqk(host0, gpu_out, fam_seed):
    """The oracle's solve_cqk (1 thread) on the same first instance."""
    import oracle

    oracle.build()
    d, a, b, l, u, r = host0
    t0 = time.perf_counter()
    out = oracle.solve_cqk(d, a, b, l, u, r, fixing=True, want_x=False)
    dt = time.perf_counter() - t0
    assert out["status"] == 0
    lam_g = gpu_out["lam"]
    parity = {"instance": fam_seed, "lam_gpu": lam_g, "lam_cpu": out["lam"],
              "lam_rel": abs(lam_g - out["lam"]) / max(1.0, abs(out["lam"])),
              "iterations_gpu": gpu_out["iterations"], "iterations_cpu": out["iterations"],
              "phi_evals_gpu": gpu_out["phi_evals"], "phi_evals_cpu": out["phi_evals"],
              "fixed_count_gpu": gpu_out["fixed_count"], "fixed_count_cpu": out["fixed_count"]}
    n = d.size
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle solve_cqk (C restatement of newton.py:209-342, fixing, 1 thread) on the "
                      f"whole first instance ({fam_seed}, n={n}, the same r); {dt:.2f} s"}, parity


# ------------------------------------------------------------------ GPU arm: C3
def run_c3(args, cfg, world, rank, local):
    import torch

    import paper_2603_15910_b200 as P

    n = args.n or cfg["n"]
    insts = cfg["instances"]
    config = bench_config("c3", cfg, world, args.n)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        dev, rs, host0, (lo, hi) = cqk_instances(cfg, n, world, rank, local)
    n_local = hi - lo
    if world > 1:
        from paper_2603_15910_b200 import distributed as D

        solvers = [D.ShardedCQK(d, r, n_total=n, offset=lo) for d, r in zip(dev, rs)]
        solve = lambda i: solvers[i].solve(variant=args.variant)  # noqa: E731
    else:
        cinst = [P.CqkInstance(*d, r=r) for d, r in zip(dev, rs)]
        fn = P.solve_cqk if args.variant == "solve" else P.jacobi_solve
        solve = lambda i: fn(cinst[i])  # noqa: E731

    def step(k):
        out = solve(k % len(insts))
        assert out.status is P.Status.SOLVED
        return {"device_ms": out.stats["device_ms"], "bytes_model": out.stats["bytes_model"],
                "lam": out.lam, "iterations": out.iterations, "phi_evals": out.phi_evals,
                "fixed_count": out.fixed_count, "inst": k % len(insts)}

    # every rank's first sharded solve spins on its peers' mailboxes (4 s
    # timeout): start the warm-up together
    barrier(world)
    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            step(k)
        ms, outs, clocks = Timed(world, local, stream).run(args.steps, step)
        h = P._native.handle(local)
        read_peak, _ = h.read_peak(dev[0])
    value = n * args.steps / (ms / 1e3)
    traffic, alg = ncu_traffic()
    tsrc = None
    if traffic is not None:
        if world > 1:  # per shard: the N=1 DRAM/algorithmic ratio on this rank's bytes
            traffic = traffic / alg * statistics.mean(o["bytes_model"] for o in outs)
            tsrc = f"{os.path.relpath(NCU_SOLVE, ROOT)} (one-GPU ncu --set full), scaled to this shard"
        else:
            tsrc = f"{os.path.relpath(NCU_SOLVE, ROOT)} (ncu --set full of this kernel, {insts[0][0]} seed {insts[0][1]})"
    rl = roofline(outs, world, read_peak, "cqk_tma_kernel<true> (persistent TMA-pipelined solve, 1 launch/solve)",
                  traffic)
    rl["traffic_source"] = tsrc

    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_cqk(args, world, rank, stream, dev, rs, host0, solvers if world > 1 else None, n, n_local)

    results = []
    for i, (fam, seed) in enumerate(insts):
        o = [x for x in outs if x["inst"] == i]
        if o:
            results.append({"instance": f"{fam}:seed{seed}", "lam": o[0]["lam"],
                            "iterations": o[0]["iterations"], "phi_evals": o[0]["phi_evals"],
                            "fixed_count": o[0]["fixed_count"],
                            "ms_min": min(x["device_ms"] for x in o)})
    cpu = parity = None
    if rank == 0 and not args.no_cpu:
        first = next(x for x in outs if x["inst"] == 0)
        cpu, parity = cpu_baseline_cqk(host0, first, f"{insts[0][0]}:seed{insts[0][1]}")
    barrier(world)
    if rank == 0:
        line = {
            "metric": cfg["metric"], "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "config": config, "roofline": rl, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks, "gpu_launches": args.steps, "results": results, "parity": parity,
            "solve": {"variant": args.variant, "n_local": n_local,
                      "median_ms_per_instance": statistics.median(r["ms_min"] for r in results)},
        }
        print(json.dumps(line), flush=True)


def e2e_cqk(args, world, rank, stream, dev, rs, host0, solvers, n, n_local):
    """The metric end to end through the public API: pinned host inputs,
    H2D + solve + D2H of x inside every timed step (first instance)."""
    import torch

    import paper_2603_15910_b200 as P

    if world > 1:
        host = [t.cpu().pin_memory().numpy() for t in dev[0]]
        xh = torch.empty(n_local, dtype=torch.float64, pin_memory=True).numpy()
        s = solvers[0]
        barrier(world)  # pinning takes rank-dependent time; the solves exchange in-kernel
        with torch.cuda.stream(stream):
            for _ in range(2):
                assert s.solve_host(host, xh).status is P.Status.SOLVED
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            barrier(world)
            e0.record(stream)
            for _ in range(args.e2e_steps):
                assert s.solve_host(host, xh).status is P.Status.SOLVED
            e1.record(stream)
            torch.cuda.synchronize()
        ems = reduce_max(e0.elapsed_time(e1) / args.e2e_steps, world)
        return {"value": n / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 5 * 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": ems,
                "api": "ShardedCQK.solve_host (each rank: its shard from pinned host memory)"}
    from paper_2603_15910_b200.pipeline import SolvePipeline

    pinned = [torch.from_numpy(v).pin_memory() for v in host0[:5]]
    inst_h = P.CqkInstance(*[t.numpy() for t in pinned], r=rs[0])

    def seq_ms():
        with torch.cuda.stream(stream):
            for _ in range(3):  # the caching host allocator settles on two pinned x blocks
                out = P.solve_cqk(inst_h)
                del out
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
            q = collections.deque()
            for _ in range(steps):
                q.append(pipe.submit(inst_h))
                if len(q) > depth:
                    assert q.popleft().result().status is P.Status.SOLVED
            while q:
                assert q.popleft().result().status is P.Status.SOLVED

        with SolvePipeline(depth=depth) as pipe:
            run(3 * depth, pipe)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run(args.e2e_steps, pipe)
            for s_ in pipe.streams:
                stream.wait_stream(s_)
            e1.record(stream)
            torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.e2e_steps

    ms_seq = seq_ms()
    ms_pipe = pipe_ms(2)
    return {"value": n / (ms_pipe / 1e3), "unit": UNIT, "h2d_bytes_per_step": 5 * 8 * n,
            "d2h_bytes_per_step": 8 * n, "ms_per_step": ms_pipe,
            "api": "SolvePipeline(depth=2).submit -> solve_cqk (first instance, pinned host arrays)",
            "sequential": {"value": n / (ms_seq / 1e3), "ms_per_step": ms_seq,
                           "api": "solve_cqk, one call after another"}}


# ------------------------------------------------------------------ GPU arm: C4 / C5
def host_normals(seed, offset_draws, count):
    """Normals of the simplex-n01 stream from draw `offset_draws` (random access)."""
    import paper_2603_15910_b200 as P

    g = P.instances.Xoshiro256pp(seed)
    g.pos = offset_draws
    return g.normal(count)


def run_c4(args, cfg, world, rank, local):
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200.distributed import shard_bounds

    n = args.n or cfg["n"]
    config = bench_config("c4", cfg, world, args.n)
    lo, hi = shard_bounds(n, world, rank)
    stream = torch.cuda.Stream()
    yh = host_normals(cfg["seed"], 2 * lo, hi - lo)  # y[lo:hi] of gen_simplex_y (2 draws each)
    zeros = reduce_max(float((yh == 0).sum()), world)
    assert zeros == 0, "an exact zero would redraw the whole vector (instances.py:78-86)"
    with torch.cuda.stream(stream):
        y = torch.from_numpy(yh).cuda()
        if world > 1:
            from paper_2603_15910_b200 import distributed as D

            comm = D.Communicator(P._native.handle(local), rank, world)
            proj = D.ShardedProjection(comm, y, n)
            solve = lambda: proj.solve(cfg["r"], l1=True)  # noqa: E731
        else:
            solve = lambda: P.simplex.project_l1_outcome(y, cfg["r"])  # noqa: E731

        def step(k):
            out = solve()
            return {"device_ms": out.stats["device_ms"], "bytes_model": out.stats["bytes_model"],
                    "lam": out.lam, "iterations": out.iterations, "phi_evals": out.phi_evals}

        barrier(world)
        for k in range(args.warmup):
            step(k)
        ms, outs, clocks = Timed(world, local, stream).run(args.steps, step)
        read_peak, _ = P._native.handle(local).read_peak([y])
    value = n * args.steps / (ms / 1e3)
    rl = roofline(outs, world, read_peak, "spx_tma_kernel<true> (persistent l1 projection, 1 launch/solve)")
    e2e = None
    if args.e2e_steps > 0:
        yp = torch.from_numpy(yh).pin_memory()
        with torch.cuda.stream(stream):
            if world > 1:
                run = lambda: proj.solve_host(yp.numpy(), cfg["r"], l1=True)  # noqa: E731
            else:
                run = lambda: P.project_l1(yp.numpy(), cfg["r"])  # noqa: E731
            barrier(world)
            run()
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                run()
            torch.cuda.synchronize()
            ems = reduce_max((time.perf_counter() - t0) * 1e3 / args.e2e_steps, world)
        e2e = {"value": n / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n, "ms_per_step": ems,
               "api": "project_l1(numpy y) per rank shard (host clock: the call returns after its D2H)"}
    cpu = None
    if rank == 0 and not args.no_cpu:
        import oracle

        oracle.build()
        m = min(10**8, yh.size)
        t0 = time.perf_counter()
        ref = oracle.project_l1(yh[:m], cfg["r"])
        dt = time.perf_counter() - t0
        cpu = {"value": m / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"oracle project_l1 (C restatement of simplex.py:311-333, 1 thread) on the first "
                         f"{m} elements of the same y; {dt:.2f} s (lam {ref['lam']})"}
    barrier(world)
    if rank == 0:
        print(json.dumps({
            "metric": cfg["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA, "config": config,
            "roofline": rl, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": args.steps,
            "results": [{"instance": config["instances"][0], "lam": outs[0]["lam"],
                         "iterations": outs[0]["iterations"], "phi_evals": outs[0]["phi_evals"]}],
        }), flush=True)


def run_c5(args, cfg, world, rank, local):
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200.distributed import shard_bounds

    rows = args.n or cfg["rows"]
    cols = cfg["cols"]
    config = bench_config("c5", cfg, world, args.n)
    lo, hi = shard_bounds(rows, world, rank)
    stream = torch.cuda.Stream()
    Yh = host_normals(cfg["seed"], 2 * lo * cols, (hi - lo) * cols).reshape(hi - lo, cols)
    zeros = reduce_max(float((Yh == 0).sum()), world)
    assert zeros == 0
    with torch.cuda.stream(stream):
        Y = torch.from_numpy(Yh).cuda()

        def step(k):
            X, lam, its, st = P.project_simplex_rows(Y, cfg["r"])
            return {"device_ms": st["device_ms"], "bytes_model": st["bytes_model"], "lam0": lam}

        for k in range(args.warmup):
            step(k)
        ms, outs, clocks = Timed(world, local, stream).run(args.steps, step)
        lam_dev = outs[-1]["lam0"]
        read_peak, _ = P._native.handle(local).read_peak([Y.view(-1)])
    n = rows * cols
    value = n * args.steps / (ms / 1e3)
    rl = roofline(outs, world, read_peak, "spx_rows_tma_kernel<4,4,8> (warp per row, bulk-copy rings, 1 launch/step)")
    e2e = None
    if args.e2e_steps > 0:
        Yp = torch.from_numpy(Yh).pin_memory().numpy()
        with torch.cuda.stream(stream):
            P.project_simplex_rows(Yp, cfg["r"])
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                P.project_simplex_rows(Yp, cfg["r"])
            ems = reduce_max((time.perf_counter() - t0) * 1e3 / args.e2e_steps, world)
        e2e = {"value": n / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n, "ms_per_step": ems,
               "api": "project_simplex_rows(numpy Y) per rank's rows (host clock: returns after its D2H)"}
    cpu = parity = None
    if rank == 0 and not args.no_cpu:
        import oracle

        oracle.build()
        m = min(16384, hi - lo)
        t0 = time.perf_counter()
        _, lam_c, _, bad = oracle.project_simplex_rows(Yh[:m], cfg["r"], threads=1)
        dt = time.perf_counter() - t0
        assert bad == 0
        lg = lam_dev[:m].cpu().numpy()
        parity = {"rows_checked": m, "lam_max_rel": float(np.max(np.abs(lg - lam_c) / np.maximum(1, np.abs(lam_c))))}
        cpu = {"value": m * cols / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"oracle newton_project_simplex per row (1 thread) on the first {m} rows of the "
                         f"same Y; {dt:.2f} s"}
    barrier(world)
    if rank == 0:
        print(json.dumps({
            "metric": cfg["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": config, "roofline": rl, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": args.steps, "parity": parity,
        }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--size", dest="n", type=int, default=None,
                    help="override n (C3/C4) or rows (C5) -- a smaller workload than the named config")
    ap.add_argument("--variant", default="solve", choices=["solve", "jacobi"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-budget", type=float, default=150.0, help="reference arm: stop timing after s")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world, rank, local = dist_init(args)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, args.config, cfg, world, rank)
        return
    import torch

    torch.cuda.set_device(local)
    {"c3": run_c3, "c4": run_c4, "c5": run_c5}[args.config](args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
