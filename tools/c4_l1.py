"""C4 on one B200: l1-ball projection of y ~ N(0,1), n = 1e9, r = 1 (BASELINE
configs[3] runs it across 8 GPUs; here the single-GPU number), with the
size-independent checks the full size allows: sum |x| = r to tolerance,
sign(x) = sign(y) on the support, x = sign(y) max(0, |y| + lam)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15910_b200 as P  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
t0 = time.time()
y = P.gen_simplex_y("simplex-n01", n, 1)
tg = time.time() - t0
yd = torch.from_numpy(y).cuda()
del y
for _ in range(2):
    out = P.simplex.project_l1_outcome(yd, 1.0)
ks = []
for _ in range(5):
    out = P.simplex.project_l1_outcome(yd, 1.0)
    ks.append(out.stats["device_ms"])
x = out.x
s_abs = float(x.abs().sum())
sign_ok = bool(((x == 0) | (torch.sign(x) == torch.sign(yd))).all())
xr = torch.sign(yd) * torch.clamp(yd.abs() + out.lam, min=0.0)
bits_ok = bool(torch.equal(x.view(torch.int64), xr.view(torch.int64)))  # signed zeros included
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
ms = min(ks)
print(json.dumps({"config": "C4 l1 n01 r=1 single GPU", "n": n, "kernel_ms": ms,
                  "elements_per_s": n / ms * 1e3, "phi_evals": out.phi_evals,
                  "bytes_model": out.stats["bytes_model"],
                  "GBps": out.stats["bytes_model"] / ms / 1e6,
                  "frac": out.stats["bytes_model"] / ms / 1e6 / peak,
                  "sum_abs_x_minus_r": s_abs - 1.0, "sign_ok": sign_ok,
                  "x_formula_maxdiff": float((x - xr).abs().max()), "x_formula_bitwise": bits_ok,
                  "host_gen_s": tg}))
