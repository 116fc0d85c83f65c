"""Build libemb.so in-tree with nvcc for sm_100a (B200). No GPU needed (cross-compiles).

    python -m paper_2112_02752_b200.build          # incremental
    python -m paper_2112_02752_b200.build --force  # rebuild everything

Objects go to paper_2112_02752_b200/build/, the library to paper_2112_02752_b200/lib/libemb.so.
Links the venv's NCCL (the same libnccl.so.2 torch loads) with an rpath to it. ptxas resource usage
(-Xptxas -v) is written to build/ptxas.log.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libemb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    try:
        import nvidia.nccl  # noqa: F401
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed: {cmd[-1]}")
    return r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    inc, libdir = nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "emb.h")]
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
             "-I", os.path.join(ROOT, "include"), "-I", inc] + ARCH
    # an object is reused only if the hash of (its source, every header, the flags) matches the stamp
    # written when it was compiled: file copies (snapshots to the GPU box) do not keep mtimes
    hh = hashlib.sha256(" ".join(flags).encode())
    for h in sorted(hdrs):
        hh.update(open(h, "rb").read())
    jobs = []
    objs = []
    stamps = {}
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        d = hh.copy()
        d.update(open(s, "rb").read())
        stamps[o] = d.hexdigest()
        st = o + ".sha"
        if force or not os.path.exists(o) or not os.path.exists(st) or open(st).read() != stamps[o]:
            jobs.append(([NVCC] + flags + ["-c", s, "-o", o], o))
    logs = []
    if jobs:
        for o in [o for _, o in jobs]:
            if os.path.exists(o + ".sha"):
                os.remove(o + ".sha")
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            logs = list(ex.map(_run, [c for c, _ in jobs]))
        for _, o in jobs:
            with open(o + ".sha", "w") as f:
                f.write(stamps[o])
        with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    link_stamp = hashlib.sha256("".join(stamps[o] for o in objs).encode()).hexdigest()
    lst = LIB + ".sha"
    if jobs or not os.path.exists(LIB) or not os.path.exists(lst) or open(lst).read() != link_stamp:
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + libdir, "-lcudart"])
        with open(lst, "w") as f:
            f.write(link_stamp)
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(force=a.force, verbose=True)
