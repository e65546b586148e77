"""Builds the in-tree native libraries.

* lib/libmsmb.so          -- the product: sm_100a CUDA kernels + host engine + C ABI
                             (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo)
* lib/libmsmb_fixtures.so -- seeded synthetic-input generator (plain C)
* ../oracle/liboracle.so, ../oracle/_ref/libparamd_ref.so -- the CPU checkers
  (test infrastructure; _ref only when /root/reference is present).

The CUDA runtime is linked statically so the library does not depend on the
runtime that PyTorch happens to load into the same process.
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
LIB = PKG / "lib"
OBJ = PKG / "lib" / "obj"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
CXX = shutil.which("g++") or "g++"
CC = "/usr/bin/gcc" if Path("/usr/bin/gcc").exists() else (shutil.which("gcc") or "gcc")

CU_SOURCES = ["msmb_kernels.cu", "msmb_engine.cu", "msmb_parareal.cu", "msmb_dd.cu", "msmb_slab.cu", "msmb_fft.cu",
              "msmb_direct.cu"]
CPP_SOURCES = ["msmb_geometry.cpp"]
HEADERS = ["msmb_internal.h", "msmb_kernels.cuh", "msmb_engine.cuh"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_msmb(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "msmb.h", Path(__file__)]
    jobs = []
    for s in CU_SOURCES:
        o = OBJ / (s + ".o")
        if force or _stale(o, [CSRC / s] + hdrs):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", str(CSRC / s), "-o", str(o)])
    for s in CPP_SOURCES:
        o = OBJ / (s + ".o")
        if force or _stale(o, [CSRC / s] + hdrs):
            jobs.append([CXX, "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off",
                         f"-I{CUDA_HOME / 'include'}", "-c", str(CSRC / s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1))) as ex:
        for out in ex.map(lambda c: _run(c, verbose), jobs):
            if verbose and out.strip():
                print(out)
    objs = [str(OBJ / (s + ".o")) for s in CU_SOURCES + CPP_SOURCES]
    so = LIB / "libmsmb.so"
    if force or jobs or _stale(so, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(so), *objs, "-lpthread"], verbose)
    return so


def build_fixtures(verbose: bool = False, force: bool = False) -> Path:
    LIB.mkdir(parents=True, exist_ok=True)
    so = LIB / "libmsmb_fixtures.so"
    src = CSRC / "fixtures.c"
    if force or _stale(so, [src]):
        _run([CC, "-std=gnu11", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", str(so), str(src), "-lm"],
             verbose)
    return so


def build_oracle(verbose: bool = False) -> None:
    """CPU checkers (test infrastructure).  _ref needs the reference sources."""
    targets = ["port"]
    if Path("/root/reference/proj/src").is_dir():
        targets += ["ref", "dropin"]
    _run(["make", "-s", "-C", str(ROOT / "oracle"), *targets], verbose)


def build_all(verbose: bool = False, force: bool = False) -> None:
    build_fixtures(verbose, force)
    build_msmb(verbose, force)
    build_oracle(verbose)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv, force="-f" in sys.argv)
