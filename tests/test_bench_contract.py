"""bench.py's reference arm on the CPU (it needs no GPU): the JSON line keeps
the driver's contract -- impl, metric / unit / higher_is_better identical to
the GPU arm's, cpu_baseline {value, unit, cores, kind, sample} and an e2e
object with zero copy bytes (a smaller --size keeps it to a second)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--size", "1000000",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    j = json.loads(line)
    assert j["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in j, k
    assert j["unit"] == "elements/s" and j["higher_is_better"] is True and j["value"] > 0
    cb = j["cpu_baseline"]
    assert set(("value", "unit", "cores", "kind", "sample")) <= set(cb) and cb["kind"] in ("port", "reference")
    assert cb["value"] == j["value"]
    e2e = j["e2e"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0 and e2e["value"] == j["value"]
    assert j["config"]["workload"].startswith("C3")
