"""Build libvenom.so (sm_100a) in-tree with nvcc. No JIT cache: the .so lives next to this file so
it travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libvenom.so")
# venom_api.cu (C ABI, format kernels) plus the SpMM kernel instantiations split into units that
# nvcc compiles in parallel (csrc/spmm_launch.cuh declares one launcher per unit)
SOURCES = [os.path.join(HERE, "csrc", "venom_api.cu")] + sorted(glob.glob(os.path.join(HERE, "csrc", "tu_*.cu")))
DEPS = SOURCES + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
    sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
LINK_FLAGS = [*ARCH, "-shared", "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


ABLATION_LIB = os.path.join(HERE, "libvenom_ablation.so")  # tools only (VENOM_DEBUG_FLAGS honoured)


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, ablation: bool = False, defines=(), name: str = "") -> str:
    """`defines` / `name`: a tools-only variant (e.g. VENOM_GATHER_P=8 -> libvenom_<name>.so), never
    the production library."""
    lib = ABLATION_LIB if ablation else (os.path.join(HERE, f"libvenom_{name}.so") if name else LIB)
    if not force and not needs_build(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    objdir = os.path.join(HERE, "build", "ablation" if ablation else (name or "release"))
    os.makedirs(objdir, exist_ok=True)
    extra = [*(["-DVENOM_ABLATION"] if ablation else []), *(["-Xptxas", "-v"] if verbose else []),
             *[f"-D{d}" for d in defines]]
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(os.path.basename(src))[0] + ".o")
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(d) for d in DEPS) and not force:
            continue
        procs.append((src, subprocess.Popen([nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", obj, src], cwd=HERE)))
    bad = [s for s, p in procs if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, f"nvcc {bad}")
    subprocess.check_call([nvcc(), *LINK_FLAGS, "-o", tmp, *objs], cwd=HERE)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    names = [a[len("--name="):] for a in sys.argv[1:] if a.startswith("--name=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, ablation="--ablation" in sys.argv,
                defines=defs, name=names[0] if names else ""))
