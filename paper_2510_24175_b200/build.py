"""Build libmhd.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Flags: --fmad=false (no FMA contraction: DESIGN.md R-ARITH, bitwise parity with the oracle),
-lineinfo (ncu source view), linked against the NCCL 2.28 that torch loads
(site-packages/nvidia/nccl)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmhd.so")
SOURCES = ["mhd_kernels.cu", "mhd_ct.cu", "mhd_split.cu", "mhd_push.cu", "mhd_api.cu"]
DEPS = SOURCES + ["mhd_device.cuh", "mhd_kernels.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl wheel not found (torch's NCCL)")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    srcs = [os.path.join(CSRC, s) for s in DEPS] + [os.path.join(ROOT, "include", "mhd.h"), __file__]
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """defines: extra -D macros (tile-shape variants for A/B measurements, e.g. MHD_TY3=4)."""
    global OUT
    if out is not None:
        OUT_, OUT = OUT, out
        try:
            return build(force=True, verbose=verbose, defines=defines)
        finally:
            OUT = OUT_
    if not force and not needs_build():
        return OUT
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "--threads", "0", "-Xcompiler", "-fPIC,-O2",
           "-shared", "-I", os.path.join(ROOT, "include"), "-I", inc, *[f"-D{d}" for d in defines],
           *os.environ.get("MHD_NVCC_EXTRA", "").split(),  # (A/B builds only)
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}", "-o", OUT + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=outs[0] if outs else None,
                defines=defs))
