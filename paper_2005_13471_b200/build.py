"""Build libbsct.so (the C-ABI library of include/bsct.h) in-tree for sm_100a.

    python -m paper_2005_13471_b200.build [--force] [-v]

Each csrc/*.cu is compiled with nvcc (-gencode arch=compute_100a,code=sm_100a -O3
-lineinfo) in parallel and linked into paper_2005_13471_b200/libbsct.so (static
cudart).  Objects are cached in build/ by source/flag hash, so rebuilding after
editing one file recompiles only that file (headers invalidate everything).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "bsct")
LIB = os.path.join(PKG, "libbsct.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", f"-I{INCLUDE}", f"-I{CSRC}"]
FLAGS += os.environ.get("BSCT_NVCC_EXTRA", "").split()  # e.g. -DBSCT_NO_F32X2 for A/B variants


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _header_hash() -> str:
    h = hashlib.sha256()
    for d in (CSRC, INCLUDE):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cuh", ".h")):
                h.update(open(os.path.join(d, f), "rb").read())
    return h.hexdigest()


def _obj_path(src: str, hh: str) -> str:
    h = hashlib.sha256()
    h.update(open(os.path.join(CSRC, src), "rb").read())
    h.update(hh.encode())
    h.update(" ".join(ARCH + FLAGS).encode())
    return os.path.join(BUILD, f"{src[:-3]}-{h.hexdigest()[:16]}.o")


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hh = _header_hash()
    srcs = _sources()
    objs = [_obj_path(s, hh) for s in srcs]

    def compile_one(pair):
        src, obj = pair
        if not force and os.path.exists(obj):
            return None
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj + ".tmp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        os.replace(obj + ".tmp", obj)
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, flush=True)
        return src

    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        done = [d for d in ex.map(compile_one, zip(srcs, objs)) if d]
    # drop cached objects of older source versions (the cache otherwise grows without bound)
    keep = set(os.path.basename(o) for o in objs) | {"libbsct.stamp"}
    for f in os.listdir(BUILD):
        if f not in keep and (f.endswith(".o") or f.endswith(".tmp")):
            try:
                os.remove(os.path.join(BUILD, f))
            except OSError:
                pass
    stamp = os.path.join(BUILD, "libbsct.stamp")
    key = "\n".join(objs)
    if done or force or not os.path.exists(LIB) or not os.path.exists(stamp) or open(stamp).read() != key:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
        open(stamp, "w").write(key)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
    sys.exit(0)
