"""Build libei.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2202_08627_b200.build [--force] [--verbose]

Objects are compiled in parallel and linked into paper_2202_08627_b200/libei.so.  The build is
keyed on a content hash of every source and header under csrc/ and include/ together with the
full nvcc command line (arch, flags, EI_NVCC_DEFS such as -DEI_TRACE / -DEI_CHECK): the hash is
written to libei.so.stamp and compiled into the library (ei_version() ends in "src:<hash>"), and
any difference rebuilds.  No CPU fallback is built.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libei.so")
STAMP = LIB + ".stamp"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "ei.h")]


def _describe():
    try:
        return subprocess.check_output(["git", "-C", ROOT, "describe", "--always", "--dirty"],
                                       stderr=subprocess.DEVNULL, text=True).strip()
    except Exception:
        return "nogit"


def _defs():
    return os.environ.get("EI_NVCC_DEFS", "").split()   # e.g. -DEI_TRACE, -DEI_CHECK (debug builds)


def source_hash() -> str:
    """16 hex digits of sha256 over the sources, headers and the nvcc command line."""
    h = hashlib.sha256()
    for p in sorted(sources() + headers()):
        h.update(os.path.relpath(p, ROOT).encode())
        h.update(open(p, "rb").read())
    # the command line with the repo root elided (the same tree hashes alike on every box)
    h.update(" ".join([NVCC] + ARCH + FLAGS + _defs()).replace(ROOT, "<root>").encode())
    return h.hexdigest()[:16]


def up_to_date() -> bool:
    try:
        return os.path.exists(LIB) and open(STAMP).read().strip() == source_hash()
    except OSError:
        return False


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sources()
    key = source_hash()
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    defs = ['-DEI_GIT_DESCRIBE="%s src:%s"' % (_describe(), key)] + _defs()
    extra = ["-Xptxas", "-v"] if verbose else []

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC] + ARCH + FLAGS + defs + extra + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = LIB + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(key + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
