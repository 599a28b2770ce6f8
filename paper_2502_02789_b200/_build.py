"""In-tree build of the native libraries (nvcc, sm_100a only).

* paper_2502_02789_b200/libspecprefill.so  <- paper_2502_02789_b200/csrc/*.cu
* spgen/libspgen.so                        <- spgen/gen.cu, spgen/probe.cu (input generator and the
                                              bench's read-stream probe; not product code)

Objects go to build/ (git-ignored); the .so files stay in-tree so gpurun ships
them to the GPU box.  Rebuilds only what changed (sources or headers newer
than the outputs).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2502_02789_b200")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libspecprefill.so")
GEN_SRC = os.path.join(ROOT, "spgen", "gen.cu")
PROBE_SRC = os.path.join(ROOT, "spgen", "probe.cu")
GEN_LIB = os.path.join(ROOT, "spgen", "libspgen.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
              "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libspecprefill.so")


def _digest(paths, extra: str = "") -> str:
    import hashlib
    h = hashlib.sha256(extra.encode())
    for p in sorted(paths):
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _newer(srcs, out, extra: str = "") -> bool:
    """Content-based staleness: rebuild when the digest of the inputs (and flags)
    differs from the one recorded next to the output."""
    stamp = out + ".sha256"
    d = _digest(srcs, extra)
    if not os.path.exists(out) or not os.path.exists(stamp) or open(stamp).read() != d:
        return True
    return False


def _stamp(srcs, out, extra: str = ""):
    with open(out + ".sha256", "w") as f:
        f.write(_digest(srcs, extra))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose: bool = False, force: bool = False) -> list[str]:
    nvcc = _nvcc()
    os.makedirs(BUILD, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    flags = " ".join(ARCH + NVCC_FLAGS)
    jobs = []
    objs = []
    for s in sources:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _newer([s] + headers, o, flags):
            jobs.append(([nvcc, *ARCH, *NVCC_FLAGS, "-Xptxas", "-v", "-c", s, "-o", o], [s] + headers, o))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for out in ex.map(lambda j: _run(j[0]), jobs):
            logs.append(out)
    for _, srcs, o in jobs:
        _stamp(srcs, o, flags)
    if force or jobs or _newer(objs, LIB):
        logs.append(_run([nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]))
        _stamp(objs, LIB)
    if force or _newer([GEN_SRC, PROBE_SRC], GEN_LIB, flags):
        logs.append(_run([nvcc, *ARCH, *NVCC_FLAGS, "-shared", GEN_SRC, PROBE_SRC, "-o", GEN_LIB]))
        _stamp([GEN_SRC, PROBE_SRC], GEN_LIB, flags)
    if verbose:
        for x in logs:
            sys.stdout.write(x)
    return logs


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print("built", LIB, GEN_LIB)
