"""Build the in-tree C-ABI shared library libca.so for sm_100a (B200).

nvcc cross-compiles here without a GPU.  FP policy: --fmad=false so the compiler
never contracts a*b+c on its own; every fused multiply-add in the kernels is an
explicit __fma_rn (reading #18).  IEEE division / sqrt (no fast-math).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libca.so")
import glob
SOURCES = [os.path.join(CSRC, "ca_api.cu")] + sorted(glob.glob(os.path.join(CSRC, "ca_sweep_*.cu")))
DEPS = SOURCES + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "ca.h"),
                                                                    os.path.abspath(__file__)]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """The NCCL bundled with torch (headers + libnccl.so.2), same image on the GPU box."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    base = os.path.join(list(spec.submodule_search_locations)[0], "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


NCCL_INC, NCCL_LIB = _nccl_dir()

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + NCCL_INC,
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Build libca.so in-tree.  `out` / `defines` (-D flags) build a tuning variant
    elsewhere (profiles/tune.py); the product library is always the in-tree one."""
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "build") if out is None else out + ".objs"
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-c", "-o", obj, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, res

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = os.path.join(HERE, "build.log") if out is None else out + ".log"
    bad = []
    with open(log, "w") as f:
        for src, obj, cmd, res in results:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                bad.append((src, res.stderr))
    if bad:
        for src, err in bad:
            sys.stderr.write(f"--- {src}\n{err[-6000:]}")
        raise RuntimeError(f"nvcc failed (see {log})")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib + ".tmp",
            *[r[1] for r in results], "-cudart", "static",
            "-Xlinker", os.path.join(NCCL_LIB, "libnccl.so.2"), "-Xlinker", "-rpath," + NCCL_LIB]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError("link failed")
    os.replace(lib + ".tmp", lib)
    if verbose:
        print(open(log).read()[-3000:])
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
