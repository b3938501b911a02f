"""Replay the reference's own test suite against the drop-in (SURVEY.md
sections 4 and 7 step 9).

  python tools/replay_reference_tests.py stage   # here: /root/reference exists
  python tools/replay_reference_tests.py run     # on the GPU box

`stage` copies /root/reference/pkg/tests/*.py, unmodified, into
oracle/_ref/reftests/ (git-ignored, so no reference source enters the
history; not gpurun-ignored, so it travels to the GPU box).  `run` executes
that suite with tests/refshim first on sys.path, so `import cqksolve` is the
B200 package (tests/refshim/cqksolve/__init__.py), and writes the per-test
outcomes to gpurun_out/refsuite.json plus a one-line summary.
"""

import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "oracle", "_ref", "reftests")
# out of scope by SURVEY.md section 2 (CLI, Condat baseline): reported apart
OUT_OF_SCOPE = ("test_cli.py", "condat", "Condat")


def stage():
    os.makedirs(DST, exist_ok=True)
    for f in sorted(os.listdir(SRC)):
        if f.endswith(".py"):
            shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))
    with open(os.path.join(DST, "pytest.ini"), "w") as f:
        f.write("[pytest]\naddopts = -p no:cacheprovider\n")
    print("staged", len([f for f in os.listdir(DST) if f.endswith(".py")]), "files into", DST)


def run():
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    report = os.path.join(out_dir, "refsuite_junit.xml")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refshim"), ROOT, DST,
                                         env.get("PYTHONPATH", "")])
    proc = subprocess.run([sys.executable, "-m", "pytest", DST, "-q", "--rootdir", DST, "-c",
                           os.path.join(DST, "pytest.ini"), f"--junitxml={report}"],
                          cwd=DST, env=env, capture_output=True, text=True)
    import xml.etree.ElementTree as ET

    cases = []
    for tc in ET.parse(report).getroot().iter("testcase"):
        status = "passed"
        msg = ""
        for kind in ("failure", "error", "skipped"):
            el = tc.find(kind)
            if el is not None:
                status = kind
                msg = (el.get("message") or "")[:300]
        name = f"{tc.get('classname')}::{tc.get('name')}"
        scope = "out_of_scope" if any(k in name or k in msg for k in OUT_OF_SCOPE) or \
            "out of scope" in msg else "in_scope"
        cases.append({"test": name, "status": status, "scope": scope, "message": msg})
    summ = {}
    for c in cases:
        key = f"{c['scope']}:{c['status']}"
        summ[key] = summ.get(key, 0) + 1
    res = {"total": len(cases), "summary": summ, "pytest_tail": proc.stdout[-600:],
           "not_passed": [c for c in cases if c["status"] != "passed"]}
    with open(os.path.join(out_dir, "refsuite.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({"total": len(cases), "summary": summ}))


if __name__ == "__main__":
    {"stage": stage, "run": run}[sys.argv[1]]()
