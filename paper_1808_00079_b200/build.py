"""In-tree build of libreforward_b200.so (planner + executor + sm_100a kernels).

    python -m paper_1808_00079_b200.build [--force] [-j N]

C++ sources compile with g++ -std=c++20, CUDA sources with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo``; everything links
into one shared library next to this file (git-ignored, shipped to the GPU
box by gpurun).  Objects are cached under build/ by source+header mtime.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ_DIR = os.path.join(ROOT, "build", "obj")
OUT = os.path.join(PKG, "libreforward_b200.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CXX = os.environ.get("CXX") or shutil.which("g++") or "g++"
CUDA_HOME = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", f"-I{INC}", f"-I{CSRC}",
            f"-I{CUDA_HOME}/include"]
NVFLAGS = ARCH + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                  f"-I{INC}", f"-I{CSRC}", "-Xptxas", "-v", "-diag-suppress", "177,550"]


def _headers():
    hs = glob.glob(os.path.join(INC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.inc"), recursive=True)
    return hs


def _sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True))
    cu = sorted(glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True))
    return cpp, cu


def _obj_path(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "__")
    return os.path.join(OBJ_DIR, rel + ".o")


def _stale(src, obj, newest_header):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or newest_header > t


def _compile(src):
    obj = _obj_path(src)
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", src, "-o", obj]
    else:
        cmd = [CXX] + CXXFLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = (r.stdout or "") + (r.stderr or "")
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{log}")
    return src, log


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    cpp, cu = _sources()
    hs = _headers()
    newest = max([os.path.getmtime(h) for h in hs] + [0.0])
    todo = [s for s in cpp + cu if force or _stale(s, _obj_path(s), newest)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            for src, log in ex.map(_compile, todo):
                if verbose and log.strip():
                    print(f"--- {os.path.relpath(src, ROOT)}\n{log}")
    objs = [_obj_path(s) for s in cpp + cu]
    if todo or not os.path.exists(OUT):
        tmp = OUT + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcuda" if False else "", "-ldl"]
        cmd = [c for c in cmd if c]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        os.replace(tmp, OUT)
    return OUT


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, jobs=a.j, verbose=a.v))


if __name__ == "__main__":
    sys.exit(main())
