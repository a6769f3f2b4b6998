"""Build the in-tree CUDA library libaaa.so (sm_100a) with nvcc."""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libaaa.so"
SOURCES = ["preprocess.cu", "scan.cu", "cull_emit.cu", "sort.cu", "raster.cu", "vtrain.cu", "backward.cu", "api.cu"]
HEADERS = ["aaa_internal.cuh", "geom.cuh", "lookback.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    root = PKG.parent
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS] + [root / "include" / "aaa.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        o = objdir / (Path(s).stem + ".o")
        objs.append(o)
        cmd = [NVCC, *FLAGS, *os.environ.get("AAA_NVCC_FLAGS", "").split(), "-c", str(CSRC / s), "-o", str(o)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + out.decode())
        if verbose and out:
            print(out.decode())
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *map(str, objs),
           "-Xcompiler", "-fPIC", "--cudart", "static"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
