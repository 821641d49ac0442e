"""Build libtps.so (sm_100a) in-tree with nvcc.  `python -m paper_2509_23241_b200.build`.

The library links the NCCL shipped in the nvidia-nccl wheel (the one torch loads) and
the static CUDA runtime; the driver API (cuTensorMapEncodeTiled) is reached through
cudaGetDriverEntryPoint, so the .so loads on a CPU-only box too (compute calls then
return TPS_E_ARCH).
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libtps.so")
SOURCES = ["gemm_sm100.cu", "elementwise.cu", "runtime.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    base = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def build(verbose: bool = False, force: bool = False, out: str | None = None, extra: list | None = None,
          objdir: str | None = None) -> str:
    """out / extra / objdir: build a variant library (e.g. -DTPS_SGD_NB=3) for experiments."""
    os.makedirs(LIBDIR, exist_ok=True)
    inc, lib = nccl_dirs()
    target = out or LIB
    odir = objdir or LIBDIR
    os.makedirs(odir, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "tps.h")]
    if not force and os.path.exists(target) and os.path.getmtime(target) >= max(os.path.getmtime(d) for d in deps):
        return target
    objs = []
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", inc]
    common += list(extra or [])
    for src in SOURCES:
        obj = os.path.join(odir, src.rsplit(".", 1)[0] + ".o")
        cmd = [nvcc()] + ARCH + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "cu"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [nvcc()] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", target] + objs + [
        "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return target


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
