"""Build libdogip.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Steps: (1) compile and run the host generator gen/gen_bhat.cpp, which writes
csrc/generated/bhat_gen.cuh from the exact reference tables; (2) nvcc every
.cu with -gencode arch=compute_100a,code=sm_100a -lineinfo; (3) link the
shared library paper_1710_09913_b200/libdogip.so (static cudart, NCCL is
dlopen'ed at run time).  Incremental: objects are rebuilt only when a source
or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libdogip.so")
GEN_OUT = os.path.join(CSRC, "generated", "bhat_gen.cuh")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CU_SOURCES = ["abi.cu", "kernels/apply.cu", "kernels/weights.cu", "kernels/vectors.cu"]


def _headers():
    out = [os.path.join(ROOT, "include", "dogip.h"), GEN_OUT]
    for d in ("host", "kernels"):
        for f in os.listdir(os.path.join(CSRC, d)):
            if f.endswith((".hpp", ".cuh", ".h")):
                out.append(os.path.join(CSRC, d, f))
    return out


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def generate(verbose=False):
    gen_src = os.path.join(CSRC, "gen", "gen_bhat.cpp")
    gen_bin = os.path.join(BUILD, "gen_bhat")
    deps = [gen_src, os.path.join(CSRC, "host", "tables.hpp")]
    if _mtime(GEN_OUT) >= max(_mtime(p) for p in deps):
        return
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(GEN_OUT), exist_ok=True)
    _run(["g++", "-O2", "-std=c++17", "-o", gen_bin, gen_src])
    _run([gen_bin, GEN_OUT])
    if verbose:
        print("generated", GEN_OUT)


def build(verbose: bool = False, force: bool = False) -> str:
    generate(verbose)
    os.makedirs(BUILD, exist_ok=True)
    hdr_t = max(_mtime(h) for h in _headers())
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                    "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace("/", "_") + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_t):
            jobs.append([NVCC] + flags + ["-c", s, "-o", o])
    if jobs:
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            logs = list(ex.map(_run, jobs))
        with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    if jobs or _mtime(LIB) < max(_mtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl"])
        if verbose:
            print("linked", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
