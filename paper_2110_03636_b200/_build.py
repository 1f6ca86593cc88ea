"""In-tree build of libhykkt.so (sm_100a) — no JIT cache, the .so travels
with the repo snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = PKG / "libhykkt.so"
INCLUDE = PKG.parent / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CPP_SOURCES = ["analyze.cpp", "host_metrics.cpp", "sysplan.cpp"]
CU_SOURCES = ["hykkt_cuda.cu"]
HEADERS = list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + [INCLUDE / "hykkt.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(map(str, cmd)) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    objs = []
    for s in CPP_SOURCES:
        src, obj = CSRC / s, OUT / (s + ".o")
        if force or _stale(obj, [src, *HEADERS]):
            _run([CXX, "-std=c++17", "-O3", "-fPIC", "-Wall", "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    for s in CU_SOURCES:
        src, obj = CSRC / s, OUT / (s + ".o")
        if force or _stale(obj, [src, *HEADERS]):
            out = _run([NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xptxas", "-v",
                        "-Xcompiler", "-fPIC", "-c", str(src), "-o", str(obj)])
            if verbose:
                print(out)
            (OUT / (s + ".ptxas.txt")).write_text(out)
        objs.append(obj)
    if force or _stale(LIB, objs):
        _run([NVCC, "-shared", *ARCH, "-cudart", "static", "-o", str(LIB), *map(str, objs)])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
