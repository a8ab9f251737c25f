"""Build libdfa.so (sm_100a) in-tree with nvcc.  No JIT cache, no torch extension:
the .so sits next to this file so it travels with the repo snapshot.

kernels.cu is compiled once as the main unit (composition kernels, launchers)
and once per table layout (kernels_m<MODE>.cu: that layout's match kernels), the
units in parallel, then linked."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("DFA_LIB") or os.path.join(HERE, "libdfa.so")
OBJDIR = os.path.join(HERE, "build")
MODE_UNITS = [f"kernels_m{m}.cu" for m in range(1, 10)]
SOURCES = ["api.cpp", "prep.cpp", "kernels.cu"] + MODE_UNITS
HEADERS = ["kernels.cuh", "prep.h", os.path.join("..", "..", "include", "dfa.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall", "-diag-suppress", "177"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    """Compile every unit (in parallel) and link `lib`.  `defines` adds -D flags
    (e.g. DFA_CHECKED for the bounds-checked build used by tools/checked_run.sh)."""
    if not force and not stale(lib):
        return lib
    tag = os.path.splitext(os.path.basename(lib))[0]
    objdir = os.path.join(OBJDIR, tag)
    os.makedirs(objdir, exist_ok=True)
    extra = [f"-D{d}" for d in defines]

    def compile_unit(src: str) -> str:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stdout + r.stderr, file=sys.stderr)
        return obj

    # biggest units first
    order = sorted(SOURCES, key=lambda f: 0 if f.startswith("kernels") else 1)
    with ThreadPoolExecutor(max(1, min(len(order), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(compile_unit, order))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
