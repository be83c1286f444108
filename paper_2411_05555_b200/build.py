"""Build the in-tree native artefacts (no JIT cache; the .so files travel with
the repo snapshot to the GPU box).

  paper_2411_05555_b200/_build/libkvsim_gpu.so  sm_100a kernels + C-ABI (product)
  paper_2411_05555_b200/_build/kvsim            C++ host CLI (kvsim run|sweep|...)
  oracle/_build/libkvsim_oracle.so              CPU oracle (test infrastructure)
  tests/_build/libkvsim_emu.so                  SIMT emulation of the kernel core (CPU tests)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
INC = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd):
    print("+", " ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)


def _csrc_deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INC, "kvsim_gpu.h")]


def build_cuda(force=False):
    os.makedirs(OUT, exist_ok=True)
    lib = os.path.join(OUT, "libkvsim_gpu.so")
    if force or _stale(lib, _csrc_deps()):
        # the lean (kvsim_sweep.cu) and full (kvsim_sweep_full.cu) kernel
        # translation units compile in parallel, then link into one library
        flags = [*ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
                 "-Xptxas", "-v", "-I" + INC]
        objs, procs = [], []
        for src in ("kvsim_sweep.cu", "kvsim_sweep_full.cu", "perfmodel.cpp"):
            obj = os.path.join(OUT, src.replace(".", "_") + ".o")
            cmd = [NVCC, *flags, "-c", "-o", obj, os.path.join(CSRC, src)]
            print("+", " ".join(cmd), file=sys.stderr)
            procs.append(subprocess.Popen(cmd))
            objs.append(obj)
        if any(p.wait() != 0 for p in procs):
            raise subprocess.CalledProcessError(1, "nvcc")
        _run([NVCC, *ARCH, "-shared", "-o", lib, *objs])
    return lib


def build_cli(force=False):
    os.makedirs(OUT, exist_ok=True)
    exe = os.path.join(OUT, "kvsim")
    src = os.path.join(CSRC, "kvsim_cli.cpp")
    if not os.path.exists(src):
        return None
    lib = build_cuda()
    if force or _stale(exe, _csrc_deps() + [lib]):
        _run(["g++", "-O3", "-std=gnu++20", "-ffp-contract=off", "-Wall", "-I" + INC, "-I" + CSRC,
              "-I/usr/local/cuda/include", "-o", exe, src, "-L" + OUT, "-lkvsim_gpu",
              "-Wl,-rpath,$ORIGIN", "-lpthread"])
    return exe


def build_oracle():
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


def build_emu(force=False):
    out = os.path.join(ROOT, "tests", "_build", "libkvsim_emu.so")
    src = os.path.join(ROOT, "tests", "emu", "kvsim_emu.cpp")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if force or _stale(out, _csrc_deps() + [src]):
        _run(["g++", "-DKVSIM_EMU", "-O2", "-std=gnu++20", "-ffp-contract=off", "-fPIC", "-shared", "-I" + INC,
              "-o", out, src, "-lpthread"])
    return out


def build_all(force=False):
    build_cuda(force)
    build_cli(force)
    build_oracle()
    build_emu(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
