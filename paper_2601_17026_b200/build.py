"""Build libcolgraph.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2601_17026_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC_DIR = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libcolgraph.so")
SOURCES = ["colgraph.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA path cannot be built")


def _inputs():
    files = [os.path.join(SRC_DIR, s) for s in SOURCES]
    files += [os.path.join(SRC_DIR, f) for f in os.listdir(SRC_DIR) if f.endswith((".cuh", ".h"))]
    files += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    return files


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    """Compile the library.  defines: extra -D flags (e.g. ("CG_LAYOUT_AOS=0",) for the
    plane-layout variant used in A/B measurements, written to another file name)."""
    if not force and os.path.exists(lib):
        mt = os.path.getmtime(lib)
        if all(os.path.getmtime(f) <= mt for f in _inputs()):
            return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-I", INCLUDE, *[f"-D{d}" for d in defines], "-o", tmp] + [os.path.join(SRC_DIR, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
    if "--debug-bounds" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_dbg.so"), defines=("CG_DEBUG_BOUNDS=1",)))
    if "--serial-scan" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_serial.so"), defines=("CG_SCAN_SERIAL=1",)))
    if "--lat-serial" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_lats.so"), defines=("CG_SCAN_LAT_GATHER=0",)))
    if "--soft-serial" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_softs.so"), defines=("CG_SOFT_GATHER=0",)))
    if "--lat-one" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_lat1.so"), defines=("CG_SCAN_LAT_ONE=1",)))
    if "--minb4" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_minb4.so"), defines=("CG_SWEEP_MINB=4",)))
    if "--col-serial" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_cols.so"), defines=("CG_SCAN_COL_GATHER=0",)))
    if "--up-late" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_uplate.so"), defines=("CG_SCAN_UP_EARLY=0",)))
    if "--scan-prof" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_prof.so"), defines=("CG_SCAN_PROF=1",)))
    if "--hplane" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_hplane.so"), defines=("CG_H_PLANE=1",)))
    if "--no-precheck" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_nopre.so"), defines=("CG_BFS_PRECHECK=0",)))
    if "--bfs-minb2" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_bfs2.so"), defines=("CG_BFS_RUN_MINB=2",)))
    if "--bfs-serial-atom" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_bfsser.so"), defines=("CG_BFS_ATOM_BATCH=0",)))
    if "--bfs-r1b2" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_bfsr1b2.so"), defines=("BFS_R=1", "CG_BFS_RUN_MINB=2")))
    if "--no-init-preload" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_noprel.so"), defines=("CG_INIT_PRELOAD=0",)))
    if "--no-fastdiv" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_nofdiv.so"), defines=("CG_FASTDIV=0",)))
    if "--soa" in sys.argv:
        print(build(force=True, lib=os.path.join(PKG, "libcolgraph_soa.so"), defines=("CG_LAYOUT_AOS=0",)))
