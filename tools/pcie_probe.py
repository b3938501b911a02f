"""Raw PCIe rates on this box: pinned host -> device and device -> host,
one stream, two streams, and both directions at once (GB/s)."""
import json
import torch

n = 100_000_000  # 800 MB
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d1():
    d.copy_(h, non_blocking=True)


def h2d2():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


def d2h1():
    h.copy_(d, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = 8 * n / 1e9
print(json.dumps({"h2d_1stream": gb / timed(h2d1) * 1e3, "h2d_2streams": 2 * gb / timed(h2d2) * 1e3,
                  "d2h_1stream": gb / timed(d2h1) * 1e3, "both_dirs_ms": timed(both),
                  "both_dirs_h2d_equiv": gb / timed(both) * 1e3}))
