"""Builds libodc.so (the C ABI of include/odc/odc.h) in-tree for sm_100a.

    python -m paper_2601_19362_b200.build        # or __graft_entry__.build()

nvcc cross-compiles here without a GPU; the .so lands in
paper_2601_19362_b200/lib/ (git-ignored, shipped to the GPU box by gpurun).
Rebuilds only when a source or header is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libodc.so")
INCLUDE = os.path.join(ROOT, "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra"]
NVFLAGS = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    hdr = sorted(glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                 + glob.glob(os.path.join(INCLUDE, "**", "*.h*"), recursive=True))
    return cu, cpp, hdr


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log):
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    log.append(" ".join(cmd) + "\n" + p.stdout)
    if p.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + p.stdout)


def build(verbose: bool = False, force: bool = False, variant: str | None = None, defines=()) -> str:
    """variant: an A/B build with extra -D defines into lib/variants/<variant>/libodc.so
    (selected at run time with ODC_LIB_PATH); the default build is lib/libodc.so."""
    cu, cpp, hdr = _sources()
    libdir = LIBDIR if variant is None else os.path.join(LIBDIR, "variants", variant)
    lib = os.path.join(libdir, "libodc.so")
    if not force and not _stale(lib, cu + cpp + hdr + [__file__]):
        return lib
    objdir = os.path.join(libdir, "obj")
    os.makedirs(objdir, exist_ok=True)
    log, objs = [], []
    inc = ["-I" + INCLUDE, "-I" + CSRC] + ["-D" + d for d in defines]
    from concurrent.futures import ThreadPoolExecutor

    jobs = []
    for src in cpp:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdr):
            jobs.append(["g++", *CXXFLAGS, *inc, "-I" + os.path.join(CUDA, "include"), "-c", src, "-o", obj])
    for src in cu:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdr):
            jobs.append([NVCC, *ARCH, *NVFLAGS, *inc, "-c", src, "-o", obj])
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(lambda c: _run(c, log), jobs))
    _run([NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", lib, *objs,
          "-Xlinker", "-rpath," + os.path.join(CUDA, "lib64"), "-lcuda"], log)
    with open(os.path.join(libdir, "build.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    # python -m paper_2601_19362_b200.build [-v] [-f] [--variant NAME DEFINE ...]
    args = sys.argv[1:]
    var, defs = None, []
    if "--variant" in args:
        i = args.index("--variant")
        var, defs = args[i + 1], [a for a in args[i + 2:] if not a.startswith("-")]
    print(build(verbose="-v" in args, force="-f" in args, variant=var, defines=defs))
