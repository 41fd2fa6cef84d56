"""In-tree build of libdbp.so (nvcc, sm_100a) -- used by __graft_entry__.build().

The library links NCCL from the nvidia-nccl wheel that torch bundles (same
soname libnccl.so.2 torch loads), with an rpath, so one NCCL is in-process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdbp.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nccl_dirs():
    try:
        import nvidia.nccl as nn  # type: ignore
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except Exception:  # pragma: no cover
        base = None
    if base and os.path.exists(os.path.join(base, "include", "nccl.h")):
        return os.path.join(base, "include"), os.path.join(base, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "dbp.h"), __file__]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build libdbp.so in-tree (or `out`, with extra -D`defines`, for tuning variants)."""
    if out is None and not force and not stale():
        return LIB
    dest = out or LIB
    inc, lib = nccl_dirs()
    tmp = dest + f".tmp{os.getpid()}"
    cmd = ["nvcc", ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           *[f"-D{d}" for d in defines], "-o", tmp] + sources() + ["-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libdbp.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, dest)
    return dest


if __name__ == "__main__":
    # python build.py [-v] [--out PATH] [-DNAME=VAL ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force=True, verbose="-v" in args, out=out, defines=defs))
