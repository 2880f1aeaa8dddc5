"""Build libskyline_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2411_14968_b200.build [--force]

Each .cu/.cpp is compiled to an object under build/ (skipped when up to
date), then linked into paper_2411_14968_b200/libskyline_b200.so so the
library travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "csrc")
OUT = os.path.join(PKG, "libskyline_b200.so")
CLI = os.path.join(PKG, "skyline-cli")
CLI_SRC = os.path.join(ROOT, "tools", "skyline_cli.cpp")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """The NCCL that torch loads (the nvidia-nccl wheel), so the process holds
    one libnccl.so.2 whichever of torch and this library loads first; the
    system NCCL otherwise."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for p in (spec.submodule_search_locations or []) if spec else []:
            if os.path.exists(os.path.join(p, "lib", "libnccl.so.2")) and os.path.exists(
                    os.path.join(p, "include", "nccl.h")):
                return p
    except (ImportError, ValueError):
        pass
    return None


NCCL_DIR = _nccl_dir()
NCCL_INC = ["-I", os.path.join(NCCL_DIR, "include")] if NCCL_DIR else []
NCCL_LINK = (["-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2", "-Xlinker",
              "-rpath=" + os.path.join(NCCL_DIR, "lib")] if NCCL_DIR else ["-lnccl"])
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include")] + NCCL_INC
CU_FLAGS = ARCH + COMMON + ["-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                            "-Xcudafe", "--diag_suppress=177", "-diag-suppress", "1444"]
SOURCES = ["kernels.cu", "kernels_dom.cu", "kernels_rand.cu", "engine.cu", "shard.cu", "small.cu", "comm.cpp", "host.cpp", "dataio.cpp", "mtjump.cpp", "angular.cpp"]
HEADERS = ["common.cuh", "kernels.cuh", "stream.cuh", "dom.cuh", "comm.hpp", "engine_impl.cuh"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "skyline_b200.h")]
    objs, jobs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer([src] + hdrs, obj):
            flags = CU_FLAGS if s.endswith(".cu") else ARCH + COMMON + ["-x", "cu"]
            if s.endswith(".cpp"):
                flags = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                         "-I", os.path.join(ROOT, "include")] + NCCL_INC
            jobs.append((s, [NVCC, *flags, "-c", src, "-o", obj]))
    # the translation units compile independently: run them side by side
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: (j[0], subprocess.run(j[1], capture_output=True, text=True)), jobs))
    for s, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
    if force or _newer(objs, OUT):
        cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-lcudart", *NCCL_LINK, "-lpthread", "-lquadmath"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    build_cli(force)
    return OUT


def build_cli(force: bool = False) -> str:
    """tools/skyline_cli.cpp -> paper_2411_14968_b200/skyline-cli (the GPU
    skyline-cli; host C++ linked against libskyline_b200.so via $ORIGIN)."""
    hdr = os.path.join(ROOT, "include", "skyline_b200.h")
    if force or _newer([CLI_SRC, hdr, OUT], CLI):
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), CLI_SRC, "-o", CLI,
               "-L", PKG, "-lskyline_b200", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("skyline-cli build failed")
    build_adapter_check(force)
    return CLI


def build_adapter_check(force: bool = False):
    """tools/adapter_check.cpp -> paper_2411_14968_b200/adapter-check: the
    drop-in adapter against the reference engine (oracle/_ref, the checker),
    built where the reference headers exist; the binary travels to the GPU."""
    ref_inc = "/root/reference/proj/include"
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libskyref.so")
    src = os.path.join(ROOT, "tools", "adapter_check.cpp")
    out = os.path.join(PKG, "adapter-check")
    if not (os.path.isdir(ref_inc) and os.path.exists(ref_so)):
        return None
    deps = [src, ref_so, OUT, os.path.join(ROOT, "adapters", "skyline_gpu.hpp")]
    if force or _newer(deps, out):
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O2", "-std=c++20", "-I", ref_inc, "-I", os.path.join(ROOT, "include"), "-I",
               os.path.join(ROOT, "adapters"), src, "-o", out, "-L", PKG, "-lskyline_b200", "-L",
               os.path.dirname(ref_so), "-lskyref", "-Wl,-rpath,$ORIGIN:$ORIGIN/../oracle/_ref"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("adapter-check build failed")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
