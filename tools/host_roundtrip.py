"""C1-sized simplex call through the C entry point vs an idle-stream event
round trip (the floor of any synchronous call).  Perf aid."""
import ctypes, time, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import _native as N
n = 10**6
y = torch.from_numpy(P.gen_simplex_y("simplex-u01", n, 1)).cuda()
h = N.handle(); x = torch.empty_like(y); o = N.make_options(None); res = N.Result()
for _ in range(50): h.lib.spx_project_f64(h.ptr, N.MEM_DEVICE, y.data_ptr(), n, 1.0, o, x.data_ptr(), res)
torch.cuda.synchronize()
K = 300
t0 = time.perf_counter()
for _ in range(K): h.lib.spx_project_f64(h.ptr, N.MEM_DEVICE, y.data_ptr(), n, 1.0, o, x.data_ptr(), res)
tc = (time.perf_counter() - t0) / K * 1e6
# raw sync cost: event record + sync on an idle stream
s = torch.cuda.Stream(); e = torch.cuda.Event()
t0 = time.perf_counter()
for _ in range(K):
    e.record(s); e.synchronize()
te = (time.perf_counter() - t0) / K * 1e6
print(json.dumps({"c_call_us": tc, "kernel_us": res.device_ms * 1e3, "idle_event_roundtrip_us": te}))
