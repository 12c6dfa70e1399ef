"""Builds the in-tree native library ``paper_2210_12924_b200/lib/libmemplan_b200.so``.

nvcc cross-compiles for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``);
there is no other architecture and no CPU fallback. The CUDA runtime is linked
statically so the library does not depend on which libcudart torch loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libmemplan_b200.so")
OBJDIR = os.path.join(ROOT, "build", "obj")

CU_SOURCES = ["mp_api.cu", "k_score.cu", "k_lifetimes.cu", "k_pairs.cu", "k_place.cu",
              "k_arena.cu", "k_lp.cu", "k_joint.cu", "k_plans.cu"]
CPP_SOURCES = ["mp_workloads.cpp", "mp_prep.cpp", "mp_parts.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _run(cmd):
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out.stdout + out.stderr)
    return out.stdout + out.stderr


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB,
          objdir: str = OBJDIR) -> str:
    """Compile and link the library. ``defines``/``lib``/``objdir`` build tuning
    variants (e.g. ``-DMP_J8_MAXT=320``) next to the product library."""
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "memplan_b200.h"))
    common = ["-O3", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
              "-Xcompiler", "-fPIC,-Wall,-fopenmp", *defines]
    objs = []
    jobs = []
    for src in CU_SOURCES + CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            extra = ["-lineinfo", "-Xptxas", "-v"] if src.endswith(".cu") else []
            jobs.append([NVCC, *ARCH, *extra, *common, "-c", s, "-o", o])
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        log = list(ex.map(_run, jobs))
    if force or _stale(lib, objs):
        log.append(_run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs,
                         "-lpthread", "-lgomp"]))
    text = "".join(log)
    if verbose:
        print(text)
    return text


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
