"""Build every native artefact in-tree (no JIT cache, so the .so files travel
with gpurun snapshots):

  paper_2201_07498_b200/libtopk_eig.so   nvcc, sm_100a only (the product)
  oracle/liboracle.so                     gcc (test infrastructure; never linked by the product)
  synthgen/libsynthgen.so                 gcc (input generators)
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2201_07498_b200")
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libtopk_eig.so")


def nccl_root() -> str:
    cands = []
    try:
        import nvidia.nccl  # type: ignore
        cands += [os.path.dirname(p) if p.endswith("__init__.py") else p
                  for p in list(getattr(nvidia.nccl, "__path__", []))]
    except Exception:
        pass
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers not found (pip nvidia-nccl)")


def sources():
    return [os.path.join(CSRC, f) for f in ("host_prep.cpp", "mem_pool.cpp", "solver.cu")]


def deps():
    return sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + \
        [os.path.join(ROOT, "include", "topk_eig.h")]


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO):
        t = os.path.getmtime(SO)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return SO
    nr = nccl_root()
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC,-fopenmp,-O3", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nr, "include"),
           *sources(), "-o", SO + ".tmp",
           "-L", os.path.join(nr, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nr, "lib"),
           "-lgomp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(SO + ".tmp", SO)
    return SO


def build_variant(out: str, defines: list[str]) -> str:
    """Dev: the library with extra -D defines (e.g. TOPK_SPMV_GQ=6) at `out`, for A/B
    runs through TOPK_LIB=<out>."""
    nr = nccl_root()
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC,-fopenmp,-O3", "-shared", *[f"-D{d}" for d in defines],
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nr, "include"),
           *sources(), "-o", out,
           "-L", os.path.join(nr, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nr, "lib"),
           "-lgomp"]
    subprocess.check_call(cmd)
    return out


def build_all(force: bool = False, verbose: bool = False):
    sys.path.insert(0, ROOT)
    import oracle
    import synthgen
    synthgen.build(force)
    oracle.build(force)
    return build_cuda(force, verbose)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv, verbose="-v" in sys.argv))
