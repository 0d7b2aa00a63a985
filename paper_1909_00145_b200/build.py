"""Build the sm_100a C-ABI library libcsc_b200.so in-tree with nvcc.

    python -m paper_1909_00145_b200.build [--force] [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, no fast-math (the
projection and the step sizes need IEEE sqrt/div).  NCCL headers come from the
torch wheel (nvidia/nccl/include); the library dlopens libnccl.so.2 only when a
context with world > 1 is created.
"""
from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcsc_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA 12.9 toolkit is required to build libcsc_b200.so")


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        base = list(nvidia.nccl.__path__)[0]
    except Exception:  # pragma: no cover
        import site
        base = None
        for sp in site.getsitepackages():
            cand = os.path.join(sp, "nvidia", "nccl")
            if os.path.isdir(cand):
                base = cand
                break
        if base is None:
            raise RuntimeError("nvidia-nccl headers not found (torch wheel)")
    inc = os.path.join(base, "include")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "csc.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in sources() + _headers())


def _flags_changed(objdir: str) -> bool:
    stamp = os.path.join(objdir, "extra_flags.txt")
    want = os.environ.get("CSC_NVCC_EXTRA", "")
    have = open(stamp).read() if os.path.exists(stamp) else ""
    if have != want:
        os.makedirs(objdir, exist_ok=True)
        with open(stamp, "w") as f:
            f.write(want)
        return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object (in parallel, only the stale ones) and link the .so."""
    if _flags_changed(os.path.join(HERE, "build")):
        force = True
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    host_cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    hdr_t = max(os.path.getmtime(p) for p in _headers())
    base = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-ccbin", host_cxx,
            "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]
    # tuning builds only (e.g. CSC_NVCC_EXTRA=-DCSC_ROLE_TIMING); the product build passes nothing
    base += [f for f in os.environ.get("CSC_NVCC_EXTRA", "").split() if f]
    if verbose:
        base.insert(1, "-Xptxas=-v")
    jobs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_t):
            jobs.append([*base, "-c", src, "-o", obj])
    from concurrent.futures import ThreadPoolExecutor
    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return subprocess.run(cmd, capture_output=not verbose, text=True)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        res = list(ex.map(run, jobs))
    for cmd, r in zip(jobs, res):
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cmd[-3]}:\n{(r.stdout or '') + (r.stderr or '')}")
    subprocess.run([nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl"], check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
