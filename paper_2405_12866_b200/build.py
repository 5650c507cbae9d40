"""Build libqfs.so (sm_100a) in-tree with nvcc.

    python -m paper_2405_12866_b200.build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; links the NCCL
bundled with torch (nvidia/nccl) with an rpath so the .so loads on the box.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqfs.so")
SOURCES = [os.path.join(CSRC, f) for f in ("qfs_kernels.cu", "qfs_resident.cu", "qfs_blocks.cu", "qfs_runtime.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "qfs_internal.h"), os.path.join(CSRC, "qfs_device.cuh"), os.path.join(ROOT, "include", "qfs.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl  # torch's bundled NCCL (namespace package)
    for p in list(nvidia.nccl.__path__):
        if os.path.exists(os.path.join(p, "include", "nccl.h")):
            return p
    raise RuntimeError("NCCL headers not found under nvidia/nccl")


LIB_DEBUG = os.path.join(HERE, "libqfs_debug.so")


def build(force: bool = False, verbose: bool = False, debug: bool = False, out: str | None = None,
          defines: list | None = None) -> str:
    """Compile libqfs.so (or, with ``debug``, libqfs_debug.so: -DQFS_DEBUG device
    bounds checks of the streamed kernels' offsets; same ABI).  ``out`` /
    ``defines``: an A/B variant of the same sources (tools/)."""
    lib = out or (LIB_DEBUG if debug else LIB)
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return lib
    nd = nccl_dir()
    libs = glob.glob(os.path.join(nd, "lib", "libnccl.so*"))
    if not libs:
        raise RuntimeError("libnccl.so not found")
    tmp = f"{lib}.tmp{os.getpid()}"
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           f"-I{os.path.join(nd, 'include')}", f"-I{os.path.join(ROOT, 'include')}",
           f"-L{os.path.join(nd, 'lib')}", f"-l:{os.path.basename(sorted(libs)[0])}",
           "-Xlinker", f"-rpath={os.path.join(nd, 'lib')}",
           *os.environ.get("QFS_NVCC_DEFINES", "").split(), *(["-DQFS_DEBUG"] if debug else []), *(defines or []),
           "-o", tmp, *SOURCES]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stdout, r.stderr)
    os.replace(tmp, lib)  # atomic: concurrent builders (one process per GPU) never see a partial file
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
