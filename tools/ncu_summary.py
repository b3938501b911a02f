"""Summarise an ncu --set full report (raw + sass pages) for profiles/."""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]


def run(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        out.append(d)
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    lines = sass.splitlines()
    stalls = collections.Counter()
    insts = collections.Counter()
    if len(lines) > 2:
        r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        h = r[0]
        iS = h.index("Warp Stall Sampling (All Samples)")
        iE = h.index("Instructions Executed")
        for row in r[1:]:
            toks = row[1].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            stalls[op] += int(row[iS] or 0)
            insts[op] += int(row[iE] or 0)
    ts, ti = sum(stalls.values()) or 1, sum(insts.values()) or 1
    top = [(o, round(100 * c / ts, 1), round(100 * insts[o] / ti, 1)) for o, c in stalls.most_common(12)]
    return {"kernels": out, "top_stall_opcodes_pct_samples_pct_insts": top}


if __name__ == "__main__":
    s = run(sys.argv[1])
    print(json.dumps(s, indent=1))
