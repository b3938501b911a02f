"""The drop-in boundary: both native libraries load without a GPU and export
every symbol their headers declare; the product path refuses to run (no CPU
fallback) when no device is visible."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+[\s\*]+(\w+)\s*\(", src, flags=re.M)))


def test_cqk_b200_exports_every_declared_symbol():
    from paper_2603_15910_b200 import _native as N

    L = N.load_library()
    names = declared("cqk_b200.h")
    assert len(names) >= 25
    missing = [s for s in names if not hasattr(L, s)]
    assert not missing, missing
    assert set(names) == set(N.EXPORTS)
    assert L.cqk_abi_version() == 1


def test_instances_exports():
    from paper_2603_15910_b200 import _native as N

    G = N.gen_library()
    names = declared("cqk_instances.h")
    assert not [s for s in names if not hasattr(G, s)]


def test_oracle_exports():
    import oracle as O

    L = O.lib()
    src = open(os.path.join(ROOT, "oracle", "cqk_oracle.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"^\s*\w+[\s\*]+(orc_\w+)\s*\(", src, flags=re.M))
    assert names and all(hasattr(L, s) for s in names)


def test_no_cpu_fallback_without_device():
    import numpy as np
    import torch

    import paper_2603_15910_b200 as P

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    inst = P.CqkInstance(d=np.ones(2), a=np.zeros(2), b=np.ones(2), l=np.zeros(2),
                         u=np.ones(2), r=1.0)
    with pytest.raises(P.NativeUnavailable):
        P.solve_cqk(inst)
    with pytest.raises(P.NativeUnavailable):
        P.newton_project_simplex(np.array([1.0, 2.0]), 1.0)


def test_library_is_sm100a():
    import subprocess

    from paper_2603_15910_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
