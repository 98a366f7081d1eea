"""In-tree build of libballmatch_b200.so (nvcc, sm_100a) — no torch JIT cache.

Run ``python -m paper_2509_01180_b200.build`` or call ``build()``.  Objects go
to ``build/``, the shared library next to this file so it travels with the repo
snapshot to the GPU box.
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
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libballmatch_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-fopenmp",
          "--expt-relaxed-constexpr", "-I", str(ROOT / "include"), "-I", str(CSRC)]
LIBS = ["-lcuda", "-lcufft", "-lgomp"]


def sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _needs(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + \
        list((ROOT / "include").glob("*.h"))
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    if _needs(obj, src):
        cmd = [NVCC, *ARCH, *CFLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
    return obj


CLI_SRC = PKG / "cli" / "ballmatch_b200_cli.cpp"
CLI_BIN = PKG / "bin" / "ballmatch-b200"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def build_cli(verbose: bool = False, force: bool = False) -> Path:
    """The ballmatch-b200 command-line front end (host C++ over the C ABI)."""
    CLI_BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [CLI_SRC, LIB, *(ROOT / "include").glob("*.h*")]
    if not force and CLI_BIN.exists() and all(d.stat().st_mtime <= CLI_BIN.stat().st_mtime for d in deps):
        return CLI_BIN
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
    cmd = [cxx, "-O2", "-std=c++20", "-Wall", "-I", str(ROOT / "include"), "-I", str(CUDA_HOME / "include"),
           str(CLI_SRC), "-o", str(CLI_BIN), "-L", str(PKG), "-lballmatch_b200", "-L", str(CUDA_HOME / "lib64"),
           "-lcudart", "-Wl,-rpath,$ORIGIN/..", "-Wl,-rpath," + str(CUDA_HOME / "lib64")]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed:\n{r.stdout}\n{r.stderr}")
    return CLI_BIN


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if force or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), *LIBS]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cli(verbose, force)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
