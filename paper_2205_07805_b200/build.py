"""Build libigs.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a),
-lineinfo for ncu source mapping, NCCL from the nvidia-nccl wheel (rpath'd)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libigs.so")
SOURCES = ["kernels.cu", "diag.cu", "api.cu", "plan.cpp"]
HEADERS = ["igs_internal.cuh", "ptx_util.cuh", "xchg.cuh", "sell_plan.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found (expected the nvidia-nccl-cu12 wheel)")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    inc, lib = nccl_dirs()
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "igs.h")]
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", inc]
    common += os.environ.get("IGS_NVCC_EXTRA", "").split()  # experiment variants (-D...)
    jobs, objs = [], []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        log = obj + ".ptxas.txt"
        if force or _stale(obj, [path] + hdrs) or (src.endswith(".cu") and not os.path.exists(log)):
            if src.endswith(".cu"):
                # -Xptxas -v: per-kernel registers / stack / spills kept next to the object
                # (tests/test_build_cpu.py checks the hot kernels have no local-memory frame)
                cmd = [NVCC, *ARCH, "-lineinfo", "-Xptxas", "-v", *common, "-c", path, "-o", obj]
            else:
                cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-I", INCLUDE, "-c", path, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if "-Xptxas" in cmd:
            with open(cmd[cmd.index("-o") + 1] + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
            return
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", lib, "-l:libnccl.so.2",
             "-Xlinker", "-rpath=" + lib])
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
