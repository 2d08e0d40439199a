"""Build the native libraries in-tree with nvcc for sm_100a (no JIT, no torch extension).

  libcodedinv.so        -- the product: csrc/*.cu behind include/codedinv.h (+ the
                           instrumentation of include/codedinv_testing.h)
  libcodedinv_probe.so  -- test-only tcgen05 probes: csrc_probe/*.cu behind include/codedinv_probe.h
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcodedinv.so")
PROBE_SRC = os.path.join(PKG, "csrc_probe")
PROBE_LIB = os.path.join(PKG, "libcodedinv_probe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"] + (["-DCI_NO_CYCLES"] if os.environ.get("CI_NO_CYCLES") else [])


def sources(d=CSRC):
    return sorted(glob.glob(os.path.join(d, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stamp(lib):
    return lib + ".flags"


def _flags_digest(extra=()):
    return hashlib.sha256(" ".join(FLAGS + list(extra)).encode()).hexdigest()


def stale(lib=LIB, srcs=None) -> bool:
    srcs = sources() if srcs is None else srcs
    if not os.path.exists(lib) or not os.path.exists(_stamp(lib)):
        return True
    if open(_stamp(lib)).read().strip() != _flags_digest():
        return True   # built with other flags (e.g. CI_NO_CYCLES)
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in srcs + headers())


def _link(srcs, lib, verbose, libs=()):
    objs = []
    for src in srcs:
        obj = os.path.join(os.path.dirname(src), os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcuda", *libs]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    with open(_stamp(lib), "w") as fh:
        fh.write(_flags_digest() + "\n")
    for o in objs:
        os.remove(o)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale(LIB, sources()):
        _link(sources(), LIB, verbose)
    if force or stale(PROBE_LIB, sources(PROBE_SRC)):
        _link(sources(PROBE_SRC), PROBE_LIB, verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
