"""Build libsa.so (sm_100a) in-tree: ``python -m paper_0905_1744_b200.build``.

One nvcc per translation unit (in parallel) compiles the CUDA kernels
(csrc/*.cu) and the host exact fallback (csrc/exact.cpp); they are linked into
``paper_0905_1744_b200/lib/libsa.so`` with the CUDA runtime linked statically, so the library does not depend on whichever
libcudart PyTorch ships.  nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib", "libsa.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    c = os.path.join(PKG, "csrc")
    return sorted(glob.glob(os.path.join(c, "*.cu"))) + sorted(glob.glob(os.path.join(c, "*.cpp")))


def headers():
    return (glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.h")) +
            [os.path.join(ROOT, "include", "sa.h")])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def _deps(src: str, seen=None) -> set:
    """The source and every local header it includes (transitively)."""
    import re
    seen = set() if seen is None else seen
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    for inc in re.findall(r'#include\s+"([^"]+)"', open(src).read()):
        for d in (os.path.dirname(src), os.path.join(ROOT, "include")):
            f = os.path.normpath(os.path.join(d, inc))
            if os.path.exists(f):
                _deps(f, seen)
                break
    return seen


def _obj(src: str) -> str:
    return os.path.join(os.path.dirname(LIB), "obj", os.path.basename(src) + ".o")


def _flags(verbose: bool):
    return [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
            "-Xptxas", "-v" if verbose else "-O3"]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit in parallel (one nvcc per file; an object
    is rebuilt when its source, a header or this script is newer), then link."""
    if not force and up_to_date():
        return LIB
    os.makedirs(os.path.join(os.path.dirname(LIB), "obj"), exist_ok=True)
    def compile_one(src):
        obj = _obj(src)
        newest = max(os.path.getmtime(f) for f in _deps(src) | {__file__})
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest:
            return src, None
        r = subprocess.run([NVCC, *_flags(verbose), "-c", src, "-o", obj + ".tmp"], capture_output=True, text=True)
        if r.returncode == 0:
            os.replace(obj + ".tmp", obj)
        return src, r

    with concurrent.futures.ThreadPoolExecutor(max_workers=len(sources())) as ex:
        results = list(ex.map(compile_one, sources()))
    for src, r in results:
        if r is None:
            continue
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"libsa build failed: {os.path.basename(src)}")
        if verbose:
            sys.stderr.write(r.stderr)
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", *[_obj(s) for s in sources()], "-ldl", "-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("libsa link failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
