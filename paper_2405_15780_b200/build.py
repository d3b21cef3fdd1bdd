"""Build libulysses_attn.so in-tree with nvcc for sm_100a.

Objects are rebuilt only when a source or header is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libulysses_attn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    purelib = sysconfig.get_paths()["purelib"]
    inc = os.path.join(purelib, "nvidia", "nccl", "include")
    lib = os.path.join(purelib, "nvidia", "nccl", "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        inc, lib = "/usr/include", "/usr/lib/x86_64-linux-gnu"
    return inc, lib


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "kernels", "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True) + \
        glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True) + [os.path.join(ROOT, "include", "ulysses_attn.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    inc, libdir = _nccl_dirs()
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(ROOT, "include"),
              "-I", CSRC]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *common, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "cu"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            sys.stdout.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out.decode())
    link = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", libdir, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath={libdir}", "-lcudart"]
    subprocess.check_call(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(name: str, defines: dict) -> str:
    """Tuning aid: build the library with extra -D macros into
    variants/lib<name>.so (for interleaved A/B timing, scripts/ab.py)."""
    inc, libdir = _nccl_dirs()
    objdir = os.path.join(HERE, "build", name)
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.join(HERE, "variants"), exist_ok=True)
    out = os.path.join(HERE, "variants", f"lib{name}.so")
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(ROOT, "include"),
              "-I", CSRC] + [f"-D{k}={v}" for k, v in defines.items()]
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *common, "-c", src, "-o", obj] + ([] if src.endswith(".cu") else ["-x", "cu"])
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        o, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + o.decode())
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs, "-L", libdir, "-l:libnccl.so.2",
                           "-Xlinker", f"-rpath={libdir}", "-lcudart"])
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        # python build.py --variant NAME KEY=VAL ...
        print(build_variant(sys.argv[2], dict(a.split("=", 1) for a in sys.argv[3:])))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
