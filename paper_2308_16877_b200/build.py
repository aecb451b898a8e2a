"""Build libhpac_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

Every .cu/.cpp under csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked into paper_2308_16877_b200/libhpac_b200.so (static cudart).
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
OBJ = PKG / "build"
LIB = PKG / "libhpac_b200.so"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-I", str(ROOT / "include"), "-I", str(CSRC),
          "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-warn-spills"]


def _sources():
    return sorted([p for p in CSRC.iterdir() if p.suffix in (".cu", ".cpp")])


def _deps():
    return [p for p in CSRC.iterdir() if p.suffix in (".cuh", ".h")] + [ROOT / "include" / "hpac_offload.h"]


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    newest_dep = max(p.stat().st_mtime for p in _deps())
    if obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, newest_dep):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-x", "cu" if src.suffix == ".cu" else "c++", "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    _build_cpp_tests(verbose)
    return LIB


def _build_cpp_tests(verbose: bool = False):
    """C++ host-API test driver (tests/cpp), linked against the in-tree .so."""
    src = ROOT / "tests" / "cpp" / "test_engine_cpp.cpp"
    exe = src.with_suffix("")
    deps = [src, ROOT / "include" / "hpac" / "hpac.hpp", LIB]
    if exe.exists() and exe.stat().st_mtime > max(p.stat().st_mtime for p in deps):
        return exe
    cmd = [NVCC, "-std=c++17", "-O2", "-x", "c++", "-I", str(ROOT / "include"), str(src),
           "-Xcompiler", "-ffp-contract=off", "-L", str(PKG), "-lhpac_b200",
           "-Xlinker", "-rpath=$ORIGIN/../../paper_2308_16877_b200", "-o", str(exe)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ test build failed:\n{r.stdout}\n{r.stderr}")
    return exe


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
