"""Build libblockeig_b200.so (sm_100a) in-tree with nvcc.

Every .cu / .cpp under csrc/ is compiled to an object under build/ and linked
into paper_2109_00485_b200/libblockeig_b200.so against cudart, cuSOLVER and
NCCL. Objects are rebuilt when their source or any header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "obj"
LIB = PKG / "libblockeig_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-pthread", "-I", str(ROOT / "include"), "-I", str(CSRC)]
CUFLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
LIBS = ["-lcudart", "-lcusolver", "-lcublas", "-lnccl", "-lpthread"]


def _headers():
    hs = list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    hdr = _headers()
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr):
        return obj
    if src.suffix == ".cu":
        cmd = [NVCC] + COMMON + CUFLAGS + ["-c", str(src), "-o", str(obj)]
    else:  # plain host C++
        cmd = [CXX, "-O3", "-std=c++20", "-fPIC", "-pthread", "-Wall", "-I", str(ROOT / "include"), "-I", str(CSRC),
               "-I", "/usr/local/cuda/include", "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return obj


def build_lib(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    cmd = [NVCC] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + ["-L/usr/local/cuda/lib64"] + LIBS
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build_lib(verbose="-v" in sys.argv))
