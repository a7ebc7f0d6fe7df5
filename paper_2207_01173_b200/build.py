"""Build libhgks.so (sm_100a) in-tree with nvcc.  No torch dependency in the library."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libhgks.so")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, os.path.join(lib, "libnccl.so.2"), lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu/libnccl.so.2", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(INCLUDE, "*.h")))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=(), extra=()) -> str:
    srcs = sources()
    out = out or LIB
    if os.sep not in out:  # bare file name: a variant next to the default library
        out = os.path.join(os.path.dirname(LIB), out)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(s) for s in srcs):
        return out
    inc, nccl_so, nccl_dir = _nccl_dirs()
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           *["-D" + d for d in defines], *extra, "-I", INCLUDE, "-I", inc, "-o", out, os.path.join(CSRC, "hgks.cu"), "-L" + nccl_dir,
           "-Xlinker", "-l:" + os.path.basename(nccl_so), "-Xlinker", "-rpath," + nccl_dir]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[5:] for a in sys.argv[1:] if a.startswith("-out=")]
    extra = [a[4:] for a in sys.argv[1:] if a.startswith("-nv=")]  # raw nvcc flags, e.g. -nv=-use_fast_math
    print(build(force=True, verbose="-v" in sys.argv, out=outs[0] if outs else None, defines=defs, extra=extra))
