"""Builds the in-tree CUDA library ``_lib/libsfb200.so`` for sm_100a with nvcc.

The library is the product: hand-written sm_100a kernels plus the C++ host
driver behind the C ABI of ``include/sforge_b200.h``.  ``--fmad=false`` keeps
every fp64 expression unfused so results are bitwise those of the reference.
"""
from __future__ import annotations

import fcntl
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libsfb200.so")
STAMP = LIB + ".sha"  # hash of the sources the library was built from
SOURCES = ["sf_kernels.cu", "sf_sweep_tma.cu", "sf_sweep2.cu", "sf_uv_tma.cu", "sf_driver.cu"]
HEADERS = ["sf_uv.cuh", "sf_device.cuh", "sf_kernels.cuh", "sf_plan.hpp", "sf_jit.hpp"]

NVCC_FLAGS = [
    "-std=c++17",
    "-O3",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--fmad=false",
    "-lineinfo",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def source_hash() -> str:
    """Hash of everything the library is built from (sources, headers, the C
    ABI header, this recipe). Content, not modification times: a snapshot of
    the tree copied to another machine keeps its prebuilt library valid."""
    h = hashlib.sha256()
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", "sforge_b200.h"), os.path.abspath(__file__)]
    for d in deps:
        with open(d, "rb") as f:
            h.update(os.path.basename(d).encode() + b"\0" + f.read())
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    """Build under an exclusive file lock (several processes -- e.g. the ranks
    of a torchrun job -- may find the library stale at once): objects go to a
    private directory, the library and its stamp are replaced atomically."""
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    with open(os.path.join(OUT_DIR, ".build.lock"), "w") as lockf:
        fcntl.flock(lockf, fcntl.LOCK_EX)
        if not force and not _stale():  # another process built it meanwhile
            return LIB
        want = source_hash()
        work = tempfile.mkdtemp(prefix=".build-", dir=OUT_DIR)
        try:
            objs = []
            log = []
            for s in SOURCES:
                obj = os.path.join(work, s.replace(".cu", ".o"))
                cmd = [_nvcc(), *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-c",
                       os.path.join(CSRC, s), "-o", obj]
                r = subprocess.run(cmd, capture_output=True, text=True)
                log.append(r.stdout + r.stderr)
                if r.returncode != 0:
                    raise RuntimeError("nvcc failed for %s:\n%s" % (s, r.stdout + r.stderr))
                objs.append(obj)
            tmp = os.path.join(work, "libsfb200.so")
            cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xlinker", "--no-undefined",
                   "-o", tmp, *objs, "-ldl"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError("nvcc link failed:\n%s" % (r.stdout + r.stderr))
            os.replace(tmp, LIB)
            with open(os.path.join(work, "stamp"), "w") as f:
                f.write(want + "\n")
            os.replace(os.path.join(work, "stamp"), STAMP)
            with open(os.path.join(OUT_DIR, "ptxas.log"), "w") as f:
                f.write("\n".join(log))
            if verbose:
                print("\n".join(log))
        finally:
            shutil.rmtree(work, ignore_errors=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
