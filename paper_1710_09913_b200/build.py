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
CU_SOURCES = (["abi.cu", "kernels/apply.cu", "kernels/weights.cu", "kernels/vectors.cu", "kernels/qp.cu"] +
              [f"kernels/apply_{d}_{p}.cu" for d in (2, 3) for p in (1, 2, 3, 4)])


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


def generate(verbose=False, gen_out=GEN_OUT, gen_args=(), build_dir=BUILD):
    gen_src = os.path.join(CSRC, "gen", "gen_bhat.cpp")
    gen_bin = os.path.join(build_dir, "gen_bhat")
    deps = [gen_src, os.path.join(CSRC, "host", "tables.hpp")]
    if _mtime(gen_out) >= max(_mtime(p) for p in deps) and not gen_args:
        return
    os.makedirs(build_dir, exist_ok=True)
    os.makedirs(os.path.dirname(gen_out), exist_ok=True)
    _run(["g++", "-O2", "-std=c++17", "-o", gen_bin, gen_src])
    _run([gen_bin, gen_out] + list(gen_args))
    if verbose:
        print("generated", GEN_OUT)


def build(verbose: bool = False, force: bool = False, variant: str = "", defines=(), gen_args=()) -> str:
    """variant != "": an experimental A/B build into _build_<variant>/ and
    libdogip_<variant>.so (load it with DOGIP_LIB=<path>)."""
    build_dir = BUILD + (f"_{variant}" if variant else "")
    lib = LIB if not variant else os.path.join(PKG, f"libdogip_{variant}.so")
    gen_out = GEN_OUT if not variant else os.path.join(build_dir, "gen", "bhat_gen.cuh")
    generate(verbose, gen_out, gen_args, build_dir)
    os.makedirs(build_dir, exist_ok=True)
    hdr_t = max(_mtime(h) for h in _headers() + [gen_out])
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                    "-I", os.path.join(ROOT, "include"), "-I", CSRC] + [f"-D{d}" for d in defines]
    if variant:
        flags += ["-DDOGIP_GEN_HEADER=\"" + gen_out + "\""]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace("/", "_") + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_t):
            jobs.append([NVCC] + flags + ["-c", s, "-o", o])
    if jobs:
        with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
            logs = list(ex.map(_run, jobs))
        with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    if jobs or _mtime(lib) < max(_mtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-ldl"])
        if verbose:
            print("linked", lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--gen-arg", dest="gen_args", action="append", default=[])
    a = ap.parse_args()
    build(verbose=True, force=a.force, variant=a.variant, defines=a.defines, gen_args=a.gen_args)
