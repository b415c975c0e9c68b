"""Build libsystec.so in-tree with nvcc for sm_100a (no JIT cache involved)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsystec.so")
# experiment builds only: extra nvcc flags (e.g. -DSYSTEC_L1_NOALLOC) into another file
EXTRA = os.environ.get("SYSTEC_NVCC_EXTRA", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v" if os.environ.get("SYSTEC_PTXAS_VERBOSE") else "-O3",
    "--expt-relaxed-constexpr",
    "-cudart", "static",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "systec.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    objs, procs = [], []
    for src in sources():      # one nvcc per translation unit, in parallel
        obj = os.path.join(CSRC, os.path.basename(src)[:-3] + (".x.o" if out else ".o"))
        cmd = [NVCC, *NVCC_FLAGS, *EXTRA, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for pr, cmd in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    tmp = lib + f".{os.getpid()}.tmp"
    # exported symbols: only the extern "C" ABI (visibility default via the macro below)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    for o in objs:
        try:
            os.remove(o)
        except OSError:
            pass
    return lib


if __name__ == "__main__":
    outp = None
    if "--out" in sys.argv:
        outp = sys.argv[sys.argv.index("--out") + 1]
    print(build(force="--force" in sys.argv, verbose=True, out=outp))
