"""Build libocean_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2503_03326_b200.build [--force] [-j N]

Objects go to paper_2503_03326_b200/build/, the shared library to
paper_2503_03326_b200/lib/libocean_b200.so (git-ignored; travels with the repo
snapshot to the GPU box). Incremental: a .cu is recompiled when it or any
header under csrc/ / include/ is newer than its object.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib", "libocean_b200.so")
API_LIB = os.path.join(PKG, "lib", "libocean_api.so")
API_TEST = os.path.join(OBJ, "test_api")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I" + os.path.join(ROOT, "include")]


def _headers():
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    newest = max(os.path.getmtime(src), _headers())
    if force or not os.path.exists(obj) or os.path.getmtime(obj) < newest:
        cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, jobs: int = 8) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl",
                                                                "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_api(force)
    return LIB


def build_api(force: bool = False) -> str:
    """The C++ drop-in API (include/ocean/*.hpp) over the C-ABI + its test program."""
    srcs = sorted(glob.glob(os.path.join(PKG, "api", "*.cpp")))
    hdrs = glob.glob(os.path.join(ROOT, "include", "ocean", "*.hpp"))
    newest = max([os.path.getmtime(f) for f in srcs + hdrs] + [os.path.getmtime(LIB)])
    if force or not os.path.exists(API_LIB) or os.path.getmtime(API_LIB) < newest:
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"),
               *srcs, "-L" + os.path.dirname(LIB), "-locean_b200", "-Wl,-rpath,$ORIGIN",
               "-o", API_LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ API build failed:\n{r.stderr}")
    test_src = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
    if os.path.exists(test_src) and (force or not os.path.exists(API_TEST) or
                                     os.path.getmtime(API_TEST) < max(newest, os.path.getmtime(test_src),
                                                                      os.path.getmtime(API_LIB))):
        cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), test_src,
               "-L" + os.path.dirname(LIB), "-locean_api", "-locean_b200",
               "-Wl,-rpath,$ORIGIN/../lib", "-o", API_TEST]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ API test build failed:\n{r.stderr}")
    return API_LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    a = ap.parse_args()
    print(build(a.force, a.j))
    sys.exit(0)
