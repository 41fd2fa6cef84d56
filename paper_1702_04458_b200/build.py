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
    """Build libdbp.so in-tree (or `out`, with extra -D`defines`, for tuning variants).
    Each .cu compiles to its own object in parallel (build_var/obj), then one link."""
    if out is None and not force and not stale():
        return LIB
    dest = out or LIB
    inc, lib = nccl_dirs()
    tag = f"{os.getpid()}.{abs(hash((dest, tuple(defines)))) % 100000}"
    objdir = os.path.join(ROOT, "build_var", "obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
             "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
             *[f"-D{d}" for d in defines]]
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + f".{tag}.o")
        objs.append(obj)
        procs.append(subprocess.Popen(["nvcc", *flags, "-c", "-o", obj, src], stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    failed = False
    for p in procs:
        o, e = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(o + e)
            failed = True
        elif verbose:
            sys.stderr.write(e)
    if failed:
        raise RuntimeError("nvcc failed building libdbp.so")
    tmp = dest + f".tmp{tag}"
    r = subprocess.run(["nvcc", ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
                        f"-Xlinker=-rpath={lib}"], capture_output=True, text=True)
    for o in objs:
        try:
            os.remove(o)
        except OSError:
            pass
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libdbp.so")
    os.replace(tmp, dest)
    return dest


if __name__ == "__main__":
    # python build.py [-v] [--out PATH] [-DNAME=VAL ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force=True, verbose="-v" in args, out=out, defines=defs))
