"""Builds the native backend, ``libmcrdl_nvl.so``, in-tree with nvcc for sm_100a.

The library is plain C ABI (include/mcrdl_nvl.h) with the CUDA runtime linked
statically and the driver VMM API resolved at run time, so it loads (and its
symbols can be checked) on a host without a GPU driver. Python binds it with
ctypes (paper_2303_08374_b200/nvl/_lib.py).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libmcrdl_nvl.so"
OBJDIR = ROOT / "build" / "obj"
SOURCES = ["comm.cu", "allreduce.cu", "exchange.cu", "exchange_api.cu", "fusion.cu", "ll.cu", "p2p.cu", "symm_x.cu", "pool.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
         "-cudart", "static", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(path).exists():
        raise RuntimeError("nvcc not found: the native backend cannot be built")
    return path


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    """Compile every CUDA source for sm_100a and link the shared library.
    trace=True builds the developer timeline variant libmcrdl_nvl_trace.so
    (-DMCRDL_TRACE; loaded when MCRDL_TRACE_LIB=1)."""
    objdir = OBJDIR.parent / "obj_trace" if trace else OBJDIR
    lib = LIBDIR / "libmcrdl_nvl_trace.so" if trace else LIB
    extra = ["-DMCRDL_TRACE"] if trace else []
    objdir.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "mcrdl_nvl.h"]
    cc = nvcc()
    jobs = []
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = objdir / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [cc, *ARCH, *FLAGS, *extra, "-Xptxas", "-v" if verbose else "-O3",
                   "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)]
            jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for cmd, res in zip(jobs, results):
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
            if verbose:
                sys.stderr.write(res.stderr)
    if force or jobs or _stale(lib, objs):
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs),
               "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                trace="--trace" in sys.argv))
