"""Build the C-ABI decode library in-tree with nvcc for sm_100a.

    python -m paper_2208_10859_b200.build [--force]

Produces ``paper_2208_10859_b200/_wvb200.so`` (static cudart, so the library
does not depend on which CUDA runtime torch loaded; device pointers and
streams are shared through the primary context) and ``_wvb200_wide.so``, the
same sources with 56-column synthesis tiles (two warp strips per K3 work
item, ``WV_K3_STRIPS=2``) for full-frame sessions
(``DecodeSession(..., tile_strips=2)``).
"""
from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["wv_select.cu", "wv_temporal.cu", "wv_idwt.cu", "wv_perspective.cu", "wv_capi.cu",
           "wv_file.cpp", "wv_encode.cu", "wv_spans.cpp"]
HEADERS = ["wv_common.cuh"]
LIB = os.path.join(HERE, "_wvb200.so")
LIB_WIDE = os.path.join(HERE, "_wvb200_wide.so")
LIBS = {LIB: (), LIB_WIDE: ("WV_K3_STRIPS=2",)}   # the shipped builds
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-diag-suppress", "177"]
# Bit-exact arithmetic (dequantisation, temporal sums, lifting) forbids FMA
# contraction; the perspective writeout's float32 geometry is approximate by
# design (+-1 LSB bar) and keeps it.
FMAD = {"wv_perspective.cu": "true"}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "wavevid_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build the shipped libraries (``LIBS``), or with ``out``/``defines`` an
    experimental variant, e.g. ``defines=["WV_K3_RP=4"]``, loaded with
    ``WV_LIB=<out>``."""
    if out or defines:
        return _build_one(out or LIB, tuple(defines), verbose)
    for lib, d in LIBS.items():
        if force or _stale(lib):
            _build_one(lib, d, verbose)
    return LIB


def _build_one(lib: str, defines, verbose: bool) -> str:
    objdir = os.path.join(HERE, "build_obj", os.path.basename(lib).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    cmds, objs = [], []
    for f in SOURCES:
        obj = os.path.join(objdir, f.rsplit(".", 1)[0] + ".o")
        cmds.append([nvcc(), *ARCH, *FLAGS, f"--fmad={FMAD.get(f, 'false')}", "-I",
                     os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines], "-c", "-o",
                     obj, os.path.join(CSRC, f)])
        objs.append(obj)
    if verbose:
        for cmd in cmds:
            print(" ".join(cmd))
    # one nvcc per source, in parallel
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(r.args)}\n{r.stderr}")
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
