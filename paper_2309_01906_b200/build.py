"""Build the native libraries in-tree (no JIT cache):

* paper_2309_01906_b200/libhpar.so  — the product (C ABI of include/hpar.h),
  nvcc for sm_100a only, cudart static, NCCL resolved at run time (dlopen).
* inputs/libhpar_inputs.so          — the seeded device input generator.

The oracle (oracle/liboracle.so) is built by oracle/oracle.py with gcc; it is
test infrastructure and shares nothing with these.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "hpar")
LIB = os.path.join(PKG, "libhpar.so")
INPUTS_LIB = os.path.join(ROOT, "inputs", "libhpar_inputs.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        return os.path.join(list(nvidia.nccl.__path__)[0], "include")
    except Exception:
        for p in ("/usr/include", "/usr/local/cuda/include"):
            if os.path.exists(os.path.join(p, "nccl.h")):
                return p
    raise RuntimeError("nccl.h not found (need the nvidia-nccl wheel headers)")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {os.path.basename(cmd[-1])}")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    incs = ["-I", INCLUDE, "-I", CSRC, "-I", _nccl_include()]
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC] + ARCH + COMMON + incs + ["-c", s, "-o", o]
            if s.endswith(".cpp"):
                cmd = [NVCC] + COMMON + incs + ["-x", "c++", "-c", s, "-o", o]
            jobs.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl", "-lpthread"])
    gsrc = os.path.join(ROOT, "inputs", "gen_device.cu")
    if force or _stale(INPUTS_LIB, [gsrc, os.path.join(INCLUDE, "hpar_inputs.h")]):
        _run([NVCC] + ARCH + COMMON + ["-I", INCLUDE, "-shared", "-cudart", "static", gsrc, "-o", INPUTS_LIB])
    if verbose:
        print("built", LIB, INPUTS_LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
