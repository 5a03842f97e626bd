"""Build libfagp_b200.so in-tree with nvcc for sm_100a.

The library is a plain C-ABI shared object (include/fagp_b200.h); no torch headers are
involved, so it builds and loads without a GPU.  Used by __graft_entry__.build() and by
`python -m paper_2403_12797_b200._build`.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libfagp_b200.so"
SOURCES = ("basis.cu", "gram.cu", "factor.cu", "predict.cu", "literal.cu", "modal.cu", "chol.cu", "fused.cu", "exact.cu", "gram_tiled.cu", "predict_tiled.cu", "host.cu")
ARCH_FLAGS = ("-gencode", "arch=compute_100a,code=sm_100a")


def nvcc_path():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfagp_b200.so")
    return cand


def _stale():
    if not LIB_PATH.exists():
        return True
    mtime = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG_DIR.parent / "include" / "fagp_b200.h"]
    return any(d.stat().st_mtime > mtime for d in deps if d.exists())


def build(force=False, verbose=False):
    """Compile every CUDA source into one shared library.  Returns its path."""
    if not force and not _stale():
        return LIB_PATH
    nvcc = nvcc_path()
    objs = []
    tmpdir = PKG_DIR / "build"
    tmpdir.mkdir(exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = tmpdir / (src + ".o")
        cmd = [nvcc, *ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", str(PKG_DIR.parent / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose and out:
            print(out, file=sys.stderr)
    tmp_lib = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp_lib), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}")
    os.replace(tmp_lib, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
