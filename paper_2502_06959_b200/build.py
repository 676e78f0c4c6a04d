"""Build libhsf.so in-tree for sm_100a (nvcc + g++).  No torch involvement."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libhsf.so")
# debug build: bounded mbarrier waits that report and trap (-DHSF_DEBUG_SYNC)
LIB_DEBUG = os.path.join(LIBDIR, "libhsf_debug.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.environ.get("NVCC", os.path.join(CUDA, "bin", "nvcc"))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function", "-fcx-limited-range"]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp", ".cuh", ".h")))


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = _sources() + [os.path.join(HERE, "..", "include", "hsf.h"), __file__]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    obj_dir = os.path.join(LIBDIR, "obj_debug" if debug else "obj")
    dflags = ["-DHSF_DEBUG_SYNC"] if debug else []
    os.makedirs(obj_dir, exist_ok=True)
    # the NVRTC prelude is embedded in the library as a raw string literal
    with open(os.path.join(CSRC, "jit_prelude.cuh")) as fh:
        prelude = fh.read()
    with open(os.path.join(obj_dir, "jit_prelude.inc"), "w") as fh:
        fh.write('R"HSFJITPRELUDE(' + prelude + ')HSFJITPRELUDE"\n')
    objs = []
    cmds = []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        if f.endswith(".cpp"):
            o = os.path.join(obj_dir, f + ".o")
            cmds.append(["g++", *CXXFLAGS, *dflags, "-I", os.path.join(HERE, "..", "include"), "-I", obj_dir,
                         "-I", os.path.join(CUDA, "include"), "-c", src, "-o", o])
            objs.append(o)
        elif f.endswith(".cu"):
            o = os.path.join(obj_dir, f + ".o")
            cmds.append([NVCC, *ARCH, *dflags, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                         "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"), "-c", src, "-o", o])
            objs.append(o)
    # compile the translation units concurrently (run.cu dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(cmds) or 1) as ex:
        results = list(ex.map(lambda c: (c, subprocess.run(c, capture_output=True, text=True)), cmds))
    for c, r in results:
        if verbose or r.returncode:
            sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"compile failed: {c[-3]}")
        # keep the ptxas report next to the objects (registers / spills / smem)
        if c[0] == NVCC:
            with open(c[-1] + ".ptxas.txt", "w") as fh:
                fh.write(r.stderr)
    tmp = lib + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-L", os.path.join(CUDA, "lib64"), "-lnvrtc",
            "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
