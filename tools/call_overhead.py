"""Host-side overhead of one public-API call (C1-sized simplex projection):
python call vs the C entry point alone vs the kernel (perf-iteration aid)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15910_b200 as P  # noqa: E402
from paper_2603_15910_b200 import _native as N  # noqa: E402

n = 10**6
y = torch.from_numpy(P.gen_simplex_y("simplex-u01", n, 1)).cuda()
for _ in range(20):
    out = P.newton_project_simplex(y, 1.0)
torch.cuda.synchronize()
K = 200
t0 = time.perf_counter()
for _ in range(K):
    out = P.newton_project_simplex(y, 1.0)
t_py = (time.perf_counter() - t0) / K
h = N.handle()
x = torch.empty_like(y)
o = N.make_options(None)
res = N.Result()
t0 = time.perf_counter()
for _ in range(K):
    h.lib.spx_project_f64(h.ptr, N.MEM_DEVICE, y.data_ptr(), n, 1.0, o, x.data_ptr(), res)
t_c = (time.perf_counter() - t0) / K
print(json.dumps({"python_call_us": 1e6 * t_py, "c_call_us": 1e6 * t_c,
                  "kernel_us": 1e3 * out.stats["device_ms"]}))
