"""Build the in-tree CUDA library `_lib/libhybridsea_b200.so` for sm_100a.

Plain nvcc, no torch extension machinery: the library exposes a C ABI
(include/hybridsea_b200.h) and is loaded with ctypes.  cudart is linked
statically so the library does not depend on which libcudart torch loaded.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libhybridsea_b200.so")
SOURCES = ["capi.cu", "fft.cu", "particles.cu", "synth.cu", "compose.cu", "init.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
              "--expt-relaxed-constexpr", "-cudart", "static"]
# particle arithmetic must round like numpy (separate IEEE mul / add); the
# kernels spell it out with __dmul_rn/__dadd_rn and this flag backs that up
PER_FILE_FLAGS = {"particles.cu": ["-fmad=false"], "init.cu": ["-fmad=false"]}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "hybridsea_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True, out: str | None = None, extra: tuple = ()) -> str:
    """Compile every csrc/*.cu (in parallel) and link the shared library.
    `out` / `extra` build an experiment variant (extra nvcc flags, e.g. -D
    switches) at another path; the product library is always `LIB`."""
    lib = out or LIB
    if not force and out is None and not extra and not needs_build():
        return LIB
    odir = os.path.dirname(lib)
    os.makedirs(odir, exist_ok=True)
    tag = os.path.basename(lib).replace(".so", "")
    jobs = []
    for src in SOURCES:
        obj = os.path.join(odir, f"{tag}_{src.replace('.cu', '.o')}")
        cmd = [nvcc(), *NVCC_FLAGS, *PER_FILE_FLAGS.get(src, []), *extra, "-I", os.path.join(ROOT, "include"),
               "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((cmd, obj))
    procs = []
    for cmd, _ in jobs:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
    bad = [cmd[-3] for (cmd, _), pr in zip(jobs, procs) if pr.wait() != 0]
    if bad:
        raise RuntimeError(f"nvcc failed on {bad}")
    objs = [o for _, o in jobs]
    tmp = lib + ".tmp"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-Xcompiler", "-fPIC", *objs, "-o", tmp]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
