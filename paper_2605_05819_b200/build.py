"""Build libhcinfer.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a).

The allocator (alloc.cpp) is compiled by g++ with -ffp-contract=off (no FMA contraction,
no fast-math) so that its float64 arithmetic is bit-identical to the oracle's.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libhcinfer.so")
BUILD = os.path.join(PKG, "_build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["api.cu", "comm.cu", "decode.cu", "prefill.cu", "repack.cu", "moe.cu", "calib.cu"]
CPP_SOURCES = ["alloc.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r.stdout + r.stderr


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib_out: str = None) -> str:
    """Compile libhcinfer.so (or, for development sweeps, a variant with extra -D defines into lib_out)."""
    build_dir = BUILD if not defines else os.path.join(BUILD, "v_" + "_".join(d.replace("=", "") for d in defines))
    lib_path = lib_out or LIB
    os.makedirs(build_dir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INC, "hcinfer.h"))
    objs = []
    jobs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC, "-c", s, "-o", o, "-std=c++17", "-O3", "-lineinfo", *ARCH,
                         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                         "-I", INC, "-I", CSRC, *dflags])
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append(["g++", "-c", s, "-o", o, "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off",
                         "-fno-fast-math", "-I", INC, "-I", CSRC])
    # independent translation units: compile them concurrently
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        log = list(ex.map(_run, jobs))
    if force or _stale(lib_path, objs):
        log.append(_run([NVCC, "-shared", "-o", lib_path, *objs, *ARCH, "-lcudart", "-ldl"]))
    out = "\n".join(x for x in log if x)
    if verbose and out:
        print(out)
    return lib_path


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("-o", dest="out", default=None)
    a = ap.parse_args()
    print(build(verbose=True, force=a.force, defines=tuple(a.defines), lib_out=a.out))
