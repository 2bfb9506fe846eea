"""Build the sm_100a shared library in-tree: paper_1804_02221_b200/_lib/libswdg_gpu.so.

nvcc cross-compiles for B200 without a GPU.  kernels_exact.cu is built with
--fmad=false (bitwise parity mode, no FMA contraction); everything else with the
default FMA contraction.  The CUDA runtime is linked statically so the .so is
self-contained on the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libswdg_gpu.so")
ROOT = os.path.dirname(PKG)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-diag-suppress=177", *os.environ.get("SWDG_NVCC_FLAGS", "").split(),
          "-I" + CSRC, "-I" + os.path.join(ROOT, "include")]

# object name -> (source, extra flags).  kernels_fast.cu is compiled once per
# degree range (SWDG_PART) so the three heavy objects build in parallel.
SOURCES = {
    "swdg_gpu": ("swdg_gpu.cu", []),
    "kernels_exact": ("kernels_exact.cu", ["--fmad=false"]),
    "kernels_common": ("kernels_common.cu", []),
    "kernels_step": ("kernels_step.cu", ["--fmad=false"]),
    "kernels_fast_p0": ("kernels_fast.cu", ["-DSWDG_PART=0", "-DSWDG_N1_LO=2", "-DSWDG_N1_HI=7"]),
    "kernels_fast_p1": ("kernels_fast.cu", ["-DSWDG_PART=1", "-DSWDG_N1_LO=8", "-DSWDG_N1_HI=11"]),
    "kernels_fast_p2": ("kernels_fast.cu", ["-DSWDG_PART=2", "-DSWDG_N1_LO=12", "-DSWDG_N1_HI=16"]),
    "kernels_mesh": ("kernels_mesh.cu", ["--fmad=false"]),
    "kernels_bench": ("kernels_bench.cu", []),
    "host_mesh": ("host_mesh.cpp", []),
}


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "swdg_gpu.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False) -> str:
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ_DIR, exist_ok=True)
    objs, cmds = [], []
    hdrs = _headers()
    for name, (src, extra) in SOURCES.items():
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(OBJ_DIR, name + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", path, "-o", obj]
            if ptxas_v:
                cmd.insert(1, "-Xptxas=-v")
            cmds.append(cmd)
    # the translation units are independent: compile them in parallel
    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(run, c) for c in cmds]:
            f.result()
    # objects of sources no longer in the build must not be linked
    for f in os.listdir(OBJ_DIR):
        if f.endswith(".o") and os.path.join(OBJ_DIR, f) not in objs:
            os.remove(os.path.join(OBJ_DIR, f))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_v="-v" in sys.argv)
