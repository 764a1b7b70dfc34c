"""Builds the sm_100a C-ABI library ``libyasps_b200.so`` in-tree.

nvcc cross-compiles for ``arch=compute_100a,code=sm_100a`` without a GPU, so the
build runs on the CPU container; the resulting ``.so`` travels to the B200 box
with the repo snapshot.  The CUDA runtime is linked statically so the library
only needs the driver at load time.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libyasps_b200.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-diag-suppress", "177", "-I", str(INCLUDE)]
SOURCES = ["ys_structure.cu", "ys_assemble.cu", "ys_solver.cu", "ys_dist.cu", "ys_contact.cu", "ys_stencil.cu", "ys_sell.cu", "ys_capi.cu"]


def _deps() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + [INCLUDE / "yasps_b200.h"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [src, *_deps(), Path(__file__)])


def _compile(src: Path, obj: Path, verbose: bool) -> str:
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        for s in SOURCES:
            src = CSRC / s
            obj = BUILD / (Path(s).stem + ".o")
            objs.append(obj)
            if force or _stale(obj, src):
                jobs.append(ex.submit(_compile, src, obj, verbose))
        logs = [j.result() for j in jobs]
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    if force or jobs or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    _build_cpp_smoke()
    return LIB


def _build_cpp_smoke():
    """The C++ facade example (include/yasps_b200.hpp) linked against the library."""
    src = PKG.parent / "tools" / "cpp_smoke.cpp"
    out = PKG.parent / "tools" / "cpp_smoke"
    if not src.exists():
        return
    if out.exists() and out.stat().st_mtime > max(src.stat().st_mtime, LIB.stat().st_mtime,
                                                   (INCLUDE / "yasps_b200.hpp").stat().st_mtime):
        return
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", str(INCLUDE), str(src), "-L", str(PKG), "-lyasps_b200",
           "-Wl,-rpath,$ORIGIN/../paper_2605_23088_b200", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cpp_smoke build failed:\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
