"""Host<->device transfer probe for the e2e leg of bench.py.

Measures pinned H2D / D2H bandwidth for one 800 MB array (one stream, and
split over several streams / both directions at once), then times one
public-API solve with host buffers split into its phases.
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ev_time(fn, stream, reps=3):
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
    nb = 8 * n
    out = {"n": n, "bytes": nb}
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        t = ev_time(lambda: d.copy_(h, non_blocking=True), s)
        out["h2d_GBs"] = nb / t / 1e6
        t = ev_time(lambda: h.copy_(d, non_blocking=True), s)
        out["d2h_GBs"] = nb / t / 1e6
    # several streams, H2D split in 4
    ss = [torch.cuda.Stream() for _ in range(4)]
    q = n // 4

    def split():
        ev = torch.cuda.Event()
        ev.record(s)
        for i, st in enumerate(ss):
            st.wait_event(ev)
            with torch.cuda.stream(st):
                d[i * q:(i + 1) * q].copy_(h[i * q:(i + 1) * q], non_blocking=True)
        for st in ss:
            e = torch.cuda.Event()
            e.record(st)
            s.wait_event(e)

    out["h2d_4streams_GBs"] = nb / ev_time(split, s) / 1e6
    # bidirectional: H2D and D2H at once
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")

    def bidir():
        ev = torch.cuda.Event()
        ev.record(s)
        ss[0].wait_event(ev)
        ss[1].wait_event(ev)
        with torch.cuda.stream(ss[0]):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(ss[1]):
            h2.copy_(d2, non_blocking=True)
        for st in ss[:2]:
            e = torch.cuda.Event()
            e.record(st)
            s.wait_event(e)

    out["bidir_GBs_total"] = 2 * nb / ev_time(bidir, s) / 1e6
    # numpy-owned pageable memory
    pg = np.ones(n)
    tp = torch.from_numpy(pg)
    with torch.cuda.stream(s):
        out["h2d_pageable_GBs"] = nb / ev_time(lambda: d.copy_(tp, non_blocking=True), s, 2) / 1e6
    # a full public-API host solve, wall clock
    import paper_2603_15910_b200 as P

    arrs = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 1)
    pinned = [torch.from_numpy(v).pin_memory() for v in arrs[:5]]
    inst = P.CqkInstance(*[t.numpy() for t in pinned], r=arrs[5])
    with torch.cuda.stream(s):
        P.solve_cqk(inst)
        torch.cuda.synchronize()
        for _ in range(3):
            t0 = time.perf_counter()
            res = P.solve_cqk(inst)
            torch.cuda.synchronize()
            out.setdefault("api_host_solve_ms", []).append(1e3 * (time.perf_counter() - t0))
        out["api_stats"] = {k: v for k, v in res.stats.items() if isinstance(v, (int, float))}
    try:
        import subprocess

        out["numa"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-1500:]
        out["pcie"] = subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
                                      "--format=csv"], capture_output=True, text=True).stdout
    except Exception:
        pass
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
