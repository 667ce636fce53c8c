"""Build recipe for the native libraries (in-tree, so the .so files travel to
the GPU box with the repo snapshot).

  paper_2201_10956_b200/libepi3cu.so   CUDA engine + C ABI (include/epi3cu.h)
  paper_2201_10956_b200/libepi3.so     C++ drop-in API (include/epi3/*.hpp) over the C ABI
  paper_2201_10956_b200/epi3_cli       `epi3 detect|verify|bench|generate` on the C++ API

sm_100a only: `-gencode arch=compute_100a,code=sm_100a`; nvcc cross-compiles
without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

LIB_CU = PKG / "libepi3cu.so"
LIB_CPP = PKG / "libepi3.so"
CLI = PKG / "epi3_cli"


def _run(cmd: list[str]) -> None:
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False) -> Path:
    srcs = [CSRC / "engine.cu", CSRC / "host.cpp"]
    deps = srcs + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "epi3cu.h"]
    if force or _stale(LIB_CU, deps):
        BUILD.mkdir(exist_ok=True)
        objs = []
        for s in srcs:
            o = BUILD / (s.stem + ".o")
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}", "-c", s, "-o", o])
            objs.append(o)
        _run([NVCC, *ARCH, "-shared", "-o", LIB_CU, *objs, "-cudart", "shared"])
    return LIB_CU


def build_cpp(force: bool = False) -> Path:
    srcs = sorted((CSRC / "api").glob("*.cpp"))
    hdrs = sorted((INCLUDE / "epi3").glob("*.hpp"))
    if not srcs:
        return LIB_CPP
    if force or _stale(LIB_CPP, srcs + hdrs + [LIB_CU]):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
              f"-I{INCLUDE}", *srcs, "-o", LIB_CPP, f"-L{PKG}", "-lepi3cu",
              f"-Wl,-rpath,$ORIGIN"])
    cli_src = CSRC / "tools" / "epi3_cli.cpp"
    if cli_src.exists() and (force or _stale(CLI, [cli_src, LIB_CPP] + hdrs)):
        _run([CXX, "-std=c++20", "-O2", "-Wall", f"-I{INCLUDE}", cli_src, "-o", CLI,
              f"-L{PKG}", "-lepi3", "-lepi3cu", f"-Wl,-rpath,$ORIGIN"])
    return LIB_CPP


def build_oracle() -> None:
    # Test infrastructure (the parity checker); see oracle/Makefile.
    _run(["make", "-s", "-f", str(ROOT / "oracle" / "Makefile"), "CC=/usr/bin/gcc",
          "CXX=/usr/bin/g++"])


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_cpp(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
