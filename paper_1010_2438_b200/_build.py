"""Build libcwcsim.so in-tree with nvcc for sm_100a (no GPU needed).

Every .cu / .cpp under csrc/ is compiled to an object in parallel, then
linked into paper_1010_2438_b200/libcwcsim.so (static CUDA runtime).
Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
(no FMA contraction anywhere in the SSA arithmetic: DESIGN.md "Rounding").
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# CWC_BUILD_TAG=<tag>: an experiment variant (objects in build_<tag>/, library
# libcwcsim_<tag>.so; tools/variant_run.py loads it); the product build has no tag
_TAG = os.environ.get("CWC_BUILD_TAG", "")
OBJ = os.path.join(HERE, "build" + ("_" + _TAG if _TAG else ""))
LIB = os.path.join(HERE, "libcwcsim" + ("_" + _TAG if _TAG else "") + ".so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
                "-I", os.path.join(ROOT, "include"), "-I", CSRC] + os.environ.get("NVCC_EXTRA", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(obj, hdrs):
    """Headers the object was compiled against (nvcc -MD output), or every
    header when the dependency file is missing."""
    dfile = obj + ".d"
    if not os.path.exists(dfile):
        return hdrs
    with open(dfile) as f:
        text = f.read().replace("\\\n", " ")
    parts = text.split(":", 1)[1].split() if ":" in text else []
    return [d for d in parts if d.startswith(ROOT) and os.path.exists(d)] or hdrs


def build(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for src in _sources():
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + _deps(obj, hdrs) + [__file__]):
            jobs.append([NVCC] + FLAGS + ["-MD", "-MF", obj + ".d", "-c", src, "-o", obj])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = [ex.submit(subprocess.run, j, capture_output=True, text=True) for j in jobs]
            for j, f in zip(jobs, futs):
                r = f.result()
                if verbose and r.stderr:
                    print(r.stderr)
                if r.returncode != 0:
                    raise RuntimeError("nvcc failed: %s\n%s" % (" ".join(j), r.stderr))
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp%d" % os.getpid()
        r = subprocess.run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose=True))
