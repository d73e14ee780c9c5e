"""Build the sm_100a shared library libmpkmeans.so in-tree with nvcc (no JIT cache).

Each .cu under csrc/ is compiled to an object in parallel with
`-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`, then linked against the NCCL that
ships with torch (rpath set, so the .so loads on the GPU box from the same image).
"""
from __future__ import annotations

import concurrent.futures as fut
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libmpkmeans.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _nccl_dir() -> str:
    import nvidia.nccl as m
    return list(m.__path__)[0]


def _flags() -> list[str]:
    nccl = _nccl_dir()
    # MPK_NVCC_EXTRA: extra flags for experiments (e.g. -DMPK_PAIR_EWG=4); not used by build()
    extra = os.environ.get("MPK_NVCC_EXTRA", "").split()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
                   "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include")] + extra


def _stale(srcs: list[str], target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) \
        + [os.path.join(ROOT, "include", "kmeans.h"), __file__]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    # experiment flags (MPK_NVCC_EXTRA) always rebuild: the library on disk may predate them
    if not force and not os.environ.get("MPK_NVCC_EXTRA") and not _stale(srcs, LIB):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()
    flags = _flags()

    def comp(src):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        cmd = [nvcc, *flags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip()):
            sys.stderr.write(r.stderr)
        return obj

    with fut.ThreadPoolExecutor(min(8, len(srcs))) as ex:
        objs = list(ex.map(comp, srcs))
    nccl = _nccl_dir()
    cmd = [nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs,
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + os.path.join(nccl, "lib"), "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
