"""One warm solve of a bench workload, for ncu captures (not a bench number)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2603_15910_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="cqk-weakly-correlated")
ap.add_argument("--n", type=int, default=10**8)
ap.add_argument("--kind", default="solve", choices=["solve", "jacobi", "simplex", "l1", "rows"])
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
if args.kind in ("solve", "jacobi"):
    d, a, b, l, u, r = P.instances.gen_cqk_arrays(args.family, args.n, 1)
    inst = P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    f = (lambda: P.solve_cqk(inst)) if args.kind == "solve" else (lambda: P.jacobi_solve(inst))
elif args.kind in ("simplex", "l1"):
    y = torch.from_numpy(P.gen_simplex_y("simplex-n01", args.n, 1)).cuda()
    f = (lambda: P.newton_project_simplex(y, 1.0)) if args.kind == "simplex" else (lambda: P.project_l1(y, 1.0))
else:
    y = torch.from_numpy(P.gen_simplex_y("simplex-n01", args.n, 1)).cuda().view(-1, 4096)
    f = lambda: P.project_simplex_rows(y, 1.0)
for _ in range(args.reps):
    out = f()
torch.cuda.synchronize()
stats = getattr(out, "stats", None) if not isinstance(out, tuple) else out[3]
print("done", stats)
os.makedirs("gpurun_out", exist_ok=True)
import json  # noqa: E402

with open(f"gpurun_out/profile_{args.kind}_stats.json", "w") as f:
    json.dump({"kind": args.kind, "family": args.family, "n": args.n, "stats": stats}, f)
