"""In-tree build of the native libraries (no JIT cache, no pip install).

* lib/libcqk_b200.so      -- CUDA kernels + C-ABI (include/cqk_b200.h), sm_100a only
* lib/libcqk_instances.so -- host instance generators (include/cqk_instances.h)

Run ``python -m paper_2603_15910_b200.build`` (or __graft_entry__.build()).
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
CUDA_LIB = os.path.join(LIBDIR, "libcqk_b200.so")
GEN_LIB = os.path.join(LIBDIR, "libcqk_instances.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction anywhere, so every product/sum in the
# element math and the scalar Newton logic rounds exactly like numpy/Python.
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-fopenmp", "-lgomp",
              "-shared", "--expt-relaxed-constexpr"]

CUDA_SOURCES = ["cqk_abi.cu"]
CUDA_DEPS = ["cqk_abi.cu", "cqk_device.cuh", "cqk_solver.cuh", "cqk_kernels.cuh", "cqk_tma.cuh", "cqk_tma_spx.cuh", "cqk_diag.cuh", "cqk_rows.cuh", "gen_kernels.cuh",
             "xoshiro_jump.h"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _cc():
    for cand in ("/usr/bin/gcc", shutil.which("gcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("gcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force=False, verbose=False):
    deps = [os.path.join(CSRC, f) for f in CUDA_DEPS] + [os.path.join(ROOT, "include", "cqk_b200.h")]
    if not force and not _stale(CUDA_LIB, deps):
        return CUDA_LIB
    os.makedirs(LIBDIR, exist_ok=True)
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(CSRC, s) for s in CUDA_SOURCES] + ["-o", CUDA_LIB]
    subprocess.check_call(cmd)
    return CUDA_LIB


def build_instances(force=False):
    src = os.path.join(CSRC, "instances.c")
    deps = [src, os.path.join(CSRC, "xoshiro_jump.h"), os.path.join(ROOT, "include", "cqk_instances.h")]
    if not force and not _stale(GEN_LIB, deps):
        return GEN_LIB
    os.makedirs(LIBDIR, exist_ok=True)
    subprocess.check_call([_cc(), "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                           "-Wall", src, "-o", GEN_LIB, "-lm"])
    return GEN_LIB


def build_all(force=False, verbose=False):
    return build_cuda(force, verbose), build_instances(force)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv, verbose="-v" in sys.argv))
