"""Write the judged ncu summaries into profiles/ (round-prefixed) from the
gpurun_out/ scratch reports.  Usage: python tools/make_profiles.py r01 [dest]
(on the GPU box: dest = gpurun_out/profiles_box, so only the small summaries
travel back)"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import run  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out")
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")
os.makedirs(dst, exist_ok=True)


def gb(s):
    v, unit = s.split()[0], s.split()[1] if len(s.split()) > 1 else ""
    f = float(v)
    return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)


for tag, rep in (("solve", "prof_solve"), ("spx", "prof_spx"), ("rows", "prof_rows")):
    path = os.path.join(src, f"{rep}_{rnd}.ncu-rep")
    if not os.path.exists(path):
        continue
    s = run(path)
    k = s["kernels"][0]
    rd, wr = gb(k["dram__bytes_read.sum"]), gb(k["dram__bytes_write.sum"])
    s["dram_bytes_per_launch"] = rd + wr
    s["source_report"] = os.path.basename(path)
    kind = {"solve": "solve", "spx": "simplex", "rows": "rows"}[tag]
    st = os.path.join(src, f"profile_{kind}_stats.json")
    if os.path.exists(st):
        rec = json.load(open(st))
        s["algorithmic_bytes_per_launch"] = rec["stats"]["bytes_model"]
        s["workload"] = {k: rec[k] for k in ("kind", "family", "n")}
        s["dram_over_algorithmic"] = (rd + wr) / rec["stats"]["bytes_model"]
    with open(os.path.join(dst, f"{rnd}_ncu_{tag}.json"), "w") as f:
        json.dump(s, f, indent=1)
launch = os.path.join(src, f"launches_{rnd}.csv")
if os.path.exists(launch):
    rows = [r for r in csv.reader(open(launch)) if len(r) > 10 and r[0] != "ID"]
    out = [{"id": r[0], "kernel": r[4], "grid": r[8], "block": r[7], "ns": r[-1]} for r in rows]
    with open(os.path.join(dst, f"{rnd}_launches.json"), "w") as f:
        json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none "
                              "python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1",
                   "launches": out}, f, indent=1)
for b in ("bench", "bench_ref"):
    p = os.path.join(src, f"{b}_{rnd}.json")
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, f"{rnd}_{b}.json"))
        continue
    p = os.path.join(src, f"{b}_{rnd}.log")  # profile_all.sh: the bench's last JSON line
    if os.path.exists(p):
        lines = [ln for ln in open(p) if ln.startswith("{")]
        if lines:
            with open(os.path.join(dst, f"{rnd}_{b}.json"), "w") as f:
                f.write(lines[-1])
print(sorted(os.listdir(dst)))
