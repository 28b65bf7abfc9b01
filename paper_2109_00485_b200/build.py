"""Build libblockeig_b200.so (sm_100a) in-tree with nvcc.

Every .cu / .cpp under csrc/ is compiled to an object under build/ and linked
into paper_2109_00485_b200/libblockeig_b200.so against cudart and cuSOLVER;
NCCL is resolved at run time (comm.cu). Objects are rebuilt when their source or any header is newer.
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
LIBS = ["-lcudart", "-lcusolver", "-lcublas", "-ldl", "-lpthread"]  # NCCL: dlopen at run time (comm.cu)


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


MIRROR_SRC = ROOT / "tests" / "cpp" / "mirror_test.cpp"
MIRROR_BIN = ROOT / "tests" / "cpp" / "mirror_test"


def build_cpp_tests(verbose: bool = False) -> Path:
    """Compile the reference-style C++ test program against the C++ mirror
    header (include/blockeig_b200.hpp) and the library."""
    lib = build_lib(verbose)
    deps = [MIRROR_SRC, ROOT / "include" / "blockeig_b200.hpp", ROOT / "include" / "blockeig_b200.h", lib]
    if MIRROR_BIN.exists() and MIRROR_BIN.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return MIRROR_BIN
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", str(ROOT / "include"), str(MIRROR_SRC),
           "-L", str(PKG), "-lblockeig_b200", "-Wl,-rpath," + str(PKG), "-o", str(MIRROR_BIN)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"mirror_test build failed:\n{r.stdout}\n{r.stderr}")
    return MIRROR_BIN


REF_TESTS = Path("/root/reference/proj/tests")
REFSUITE = ROOT / "tests" / "refsuite"
REFSUITE_BIN = REFSUITE / "bin"
REF_SUITES = ("test_kernels", "test_precond", "test_lobpcg", "test_densela", "test_csb")


def build_refsuite(verbose: bool = False) -> dict:
    """Compile the reference's OWN unit suites (/root/reference/proj/tests/test_*.cpp,
    unmodified, read in place) against the C++ mirror header: their
    #include "blockeig/*.hpp" resolve to tests/refsuite/include/blockeig/ (forwarders
    to include/blockeig_b200.hpp) and <doctest.h> to the minimal doctest shim. The
    binaries land in tests/refsuite/bin/ (git-ignored, shipped to the GPU box like
    the library). Only possible where /root/reference exists (this container);
    returns {suite: "ok" | error text}."""
    lib = build_lib(verbose)
    out = {}
    if not REF_TESTS.is_dir():
        return out
    REFSUITE_BIN.mkdir(parents=True, exist_ok=True)
    inc = REFSUITE / "include"
    deps = [ROOT / "include" / "blockeig_b200.hpp", ROOT / "include" / "blockeig_b200.h", lib, inc / "doctest.h"]
    newest_dep = max(d.stat().st_mtime for d in deps)

    def one(name):
        src = REF_TESTS / f"{name}.cpp"
        exe = REFSUITE_BIN / name
        if exe.exists() and exe.stat().st_mtime >= max(newest_dep, src.stat().st_mtime):
            return name, "ok"
        cmd = [CXX, "-std=c++20", "-O2", "-I", str(inc), "-I", str(ROOT / "include"), str(src), "-L", str(PKG),
               "-lblockeig_b200", "-Wl,-rpath," + str(PKG), "-o", str(exe)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            if exe.exists():
                exe.unlink()
            return name, (r.stderr or r.stdout)[-4000:]
        return name, "ok"

    with cf.ThreadPoolExecutor(max_workers=len(REF_SUITES)) as ex:
        for name, res in ex.map(one, REF_SUITES):
            out[name] = res
    return out


if __name__ == "__main__":
    print(build_lib(verbose="-v" in sys.argv))
