"""Builds libexitmeasure_b200.so in-tree (paper_2409_03686_b200/lib/).

nvcc cross-compiles for sm_100a only (``-gencode arch=compute_100a,
code=sm_100a``), with ``-lineinfo`` so ncu's source page maps to the .cu
files.  The FP64 mirror (walk_ref64.cu) is compiled with ``-fmad=false`` so
its arithmetic matches the reference's non-FMA gcc build bit for bit; the
production FP32 kernel keeps FMA contraction.  cudart is linked statically so
the library does not depend on which libcudart torch has already loaded.

Usage: python -m paper_2409_03686_b200.build_native [--verbose]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "lib"
LIB = OUT_DIR / "libexitmeasure_b200.so"
BUILD = PKG / "_build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", str(PKG.parent / "include")]

UNITS = [
    # (source, extra flags)
    ("walk_ref64.cu", ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"]),
    ("walk_f32.cu", ["-fmad=true", "-prec-sqrt=false", "-prec-div=false",
                     f"-DEM_BATCH_STEPS={os.environ.get('EM_BATCH_STEPS', '8')}",
                     f"-DEM_MIN_BLOCKS={os.environ.get('EM_MIN_BLOCKS', '0')}",
                     f"-DEM_ANGLE_BITS={os.environ.get('EM_ANGLE_BITS', '16')}",
                     f"-DEM_Z_BITS={os.environ.get('EM_Z_BITS', '16')}",
                     f"-DEM_TAB_WARP={os.environ.get('EM_TAB_WARP', '0')}",
                     f"-DEM_ROLL2_BLOCKS={os.environ.get('EM_ROLL2_BLOCKS', '4')}",
                     f"-DEM_ROLL2_DYN={os.environ.get('EM_ROLL2_DYN', '0')}",
                     f"-DEM_POST_STOP={os.environ.get('EM_POST_STOP', '1')}",
                     f"-DEM_TANG_K={os.environ.get('EM_TANG_K', '4')}"]),
    ("capi.cu", []),
    ("kat_curand.cu", []),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources_newer(target: Path) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    files = list(CSRC.glob("*")) + list((PKG.parent / "include").glob("*.h")) + [Path(__file__)]
    return any(f.stat().st_mtime > t for f in files)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _sources_newer(LIB):
        return LIB
    BUILD.mkdir(exist_ok=True)
    OUT_DIR.mkdir(exist_ok=True)
    nv = nvcc()
    objs = []
    for src, extra in UNITS:
        obj = BUILD / (Path(src).stem + ".o")
        cmd = [nv, "-c", str(CSRC / src), "-o", str(obj)] + ARCH + NVCC_COMMON + extra
        if verbose:
            cmd += ["-Xptxas", "-v"]
        _run(cmd, verbose)
        objs.append(str(obj))
    gobj = BUILD / "grid.o"
    _run(["g++", "-O2", "-fPIC", "-std=c++17", "-c", str(CSRC / "grid.cpp"), "-o", str(gobj)],
         verbose)
    objs.append(str(gobj))
    tmp = LIB.with_suffix(".so.tmp")
    _run([nv, "-shared", "-o", str(tmp)] + objs + ARCH + ["-cudart", "static", "-lpthread"],
         verbose)
    os.replace(tmp, LIB)
    return LIB


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and (res.stdout or res.stderr):
        print(res.stdout + res.stderr, file=sys.stderr, flush=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force or a.verbose, verbose=a.verbose))
