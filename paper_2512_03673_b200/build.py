"""Build the sm_100a shared library libconvrot_b200.so in-tree.

    python -m paper_2512_03673_b200.build [--force] [-j N]

Every translation unit under csrc/ is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo`` (tcgen05 PTX is
only legal for the arch-specific sm_100a target) into _build/, in parallel,
and linked into ``paper_2512_03673_b200/libconvrot_b200.so`` with the CUDA
runtime linked statically so the .so travels with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libconvrot_b200.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-I" + INCLUDE, "-I" + CSRC,
                     "-diag-suppress", "177"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(INCLUDE, "crt", "*.h")))


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


# next to the library (it travels with it; _build/ does not)
FLAGS_STAMP = LIB[:-3] + ".flags"


def _flags() -> str:
    """The compile flags objects are built with, without the (checkout-
    dependent) include paths; a change (e.g. a CRT_NVCC_EXTRA A/B build)
    invalidates every object."""
    return " ".join(f for f in NVCC_FLAGS + os.environ.get("CRT_NVCC_EXTRA", "").split()
                    if not f.startswith("-I"))


def _flags_changed() -> bool:
    try:
        with open(FLAGS_STAMP) as f:
            return f.read() != _flags()
    except OSError:
        return True


def needs_build() -> bool:
    if not os.path.exists(LIB) or _flags_changed():
        return True
    return _newest(_sources() + _headers() + [__file__]) > os.path.getmtime(LIB)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    hdr_time = _newest(_headers() + [__file__])
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time)):
        return obj
    extra = os.environ.get("CRT_NVCC_EXTRA", "").split()  # dev aid: A/B builds
    cmd = [nvcc()] + NVCC_FLAGS + extra + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, jobs: int = 0, verbose: bool = True) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    if _flags_changed():
        force = True
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    if verbose:
        print(f"[build] nvcc {len(srcs)} TUs for sm_100a (-j{jobs})", file=sys.stderr)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-cudart", "static", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(FLAGS_STAMP, "w") as f:
        f.write(_flags())
    if verbose:
        print(f"[build] wrote {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=0)
    args = ap.parse_args()
    build(force=args.force, jobs=args.j)
