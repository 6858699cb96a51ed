"""Build libsem.so in-tree: hand-written CUDA for sm_100a + host C++ planner,
linked against the NCCL that ships with torch (one libnccl.so.2 per process)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
SO = os.path.join(HERE, "libsem.so")
ROOT = os.path.dirname(HERE)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_SRCS = ["ax.cu", "kern.cu", "p2p.cu", "krylov.cu", "schwarz.cu", "coarse.cu", "loopback.cu", "api.cu"]
CXX_SRCS = ["plan.cpp"]


def _nccl_dirs():
    import nvidia.nccl  # torch's NCCL 2.28 (pip package)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _deps_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "sem.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def _check_spills(log: str, limit: int = 16):
    """Warn when a hot-path kernel spills: the register allocation of the Ax
    kernel is close to the residency cap and a spill costs ~20% of throughput."""
    import re
    bad = []
    for chunk in log.split("Compiling entry function")[1:]:
        name = chunk.split("'")[1]
        m = re.search(r"(\d+) bytes spill stores", chunk)
        if m and int(m.group(1)) > limit and ("ax_kernel" in name or "cg_" in name or "gs_" in name):
            bad.append((name, int(m.group(1))))
    for name, b in bad:
        print(f"WARNING: {name} spills {b} bytes", file=sys.stderr)
    return bad


def build(force: bool = False, verbose: bool = False, defines=(), variant: str | None = None) -> str:
    """Build libsem.so; with variant, a tuning build (extra -D defines) into
    _var/libsem_<variant>.so, loaded only when SEM_LIB points at it."""
    so, obj = SO, OBJ
    if variant:
        obj = os.path.join(HERE, "_var", variant)
        so = os.path.join(HERE, "_var", f"libsem_{variant}.so")
    if not force and os.path.exists(so) and os.path.getmtime(so) >= _deps_mtime():
        return so
    os.makedirs(obj, exist_ok=True)
    inc, lib = _nccl_dirs()
    nvcc = _nvcc()
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc,
              "-I", os.path.join(ROOT, "include"), *defines]
    jobs = []
    for f in CUDA_SRCS:
        out = os.path.join(obj, f + ".o")
        jobs.append([nvcc, *ARCH, *common, "-Xptxas", "-v", "-c", os.path.join(CSRC, f), "-o", out])
    for f in CXX_SRCS:
        out = os.path.join(obj, f + ".o")
        jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-I",
                     os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, f), "-o", out])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        logs = list(ex.map(run, jobs))
    with open(os.path.join(obj, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    _check_spills("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    objs = [os.path.join(obj, f + ".o") for f in CUDA_SRCS + CXX_SRCS]
    run([nvcc, *ARCH, "-shared", "-o", so + ".tmp", *objs, "-L", lib, "-l:libnccl.so.2",
         "-Xlinker", "-rpath=" + lib, "-lcudart"])
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    # python build.py [--force] [-v] [--variant NAME -DMACRO=V ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    print(build(force="--force" in args, verbose="-v" in args,
                defines=[a for a in args if a.startswith("-D")], variant=var))
