"""Build libhivc_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2008_10273_b200.build        (or __graft_entry__.build())
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libhivc_b200.so"
OBJ = PKG / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction, so float64 expressions round exactly like numpy's
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-I", str(PKG.parent / "include")]
FLAGS += os.environ.get("HIVC_NVCC_EXTRA", "").split()  # experiments (e.g. -DHIVC_FRAME_MIN_BLOCKS=12)
SOURCES = ["parse.cpp", "encode.cpp", "inpaint.cu", "recon.cu", "brox.cu", "blockgemm.cu", "decode.cu", "abi.cu"]


def _compile(src: str) -> Path:
    s = CSRC / src
    o = OBJ / (src + ".o")
    deps = [s] + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "hivc_b200.h"]
    if o.exists() and all(o.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return o
    lang = ["-x", "cu"] if s.suffix == ".cu" else ["-x", "c++"]
    cmd = [NVCC, *ARCH, *FLAGS, *lang, "-c", str(s), "-o", str(o)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    return o


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if OUT.exists() and all(OUT.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return OUT
    cmd = [NVCC, *ARCH, "-shared", "-o", str(OUT), *map(str, objs), "-lcudart", "-Xcompiler", "-pthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
