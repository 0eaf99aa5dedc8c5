"""Build libngsgd.so in-tree with nvcc for sm_100a (no torch JIT, no caches outside the repo).

Usage: python -m paper_1410_7455_b200.build   (or via __graft_entry__.build()).
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libngsgd.so")
SOURCES = ["ngsgd.cu", "nnet.cu", "gemm_tc.cu", "simple_ng.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl  # torch's bundled NCCL 2.28 (same image on the GPU box)
    return list(nvidia.nccl.__path__)[0]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "ngsgd.h"), __file__]
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return LIB
    nd = nccl_dir()
    objs = []
    jobs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if os.environ.get("NG_PTXAS_V") else "-O3",
               "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
               "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for src, cmd, p in jobs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose and out.strip():
            sys.stderr.write(out)
    link = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("link failed")
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
