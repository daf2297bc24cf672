"""Build libcafs_b200.so in-tree with nvcc (sm_100a only).

    python -m paper_2605_25040_b200.build          # incremental
    python -m paper_2605_25040_b200.build --force

Each ``csrc/*.cu`` compiles to ``build/obj/*.o`` in parallel; the objects link
into ``paper_2605_25040_b200/libcafs_b200.so`` (git-ignored, but it travels to
the GPU box with the gpurun snapshot).
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libcafs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    """The NCCL that torch ships (nvidia-nccl wheel): headers and libnccl.so.2."""
    try:
        import nvidia.nccl
        d = list(nvidia.nccl.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    except ImportError:
        pass
    return ""


NCCL = _nccl_dir()
NCCL_INC = ["-I", os.path.join(NCCL, "include")] if NCCL else []
NCCL_LINK = (["-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker",
              "-rpath=" + os.path.join(NCCL, "lib")] if NCCL else ["-lnccl"])
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _deps() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "cafs_b200.h")]


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    newest = max(os.path.getmtime(p) for p in [src] + _deps())
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *NCCL_INC, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", *NCCL_LINK]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
