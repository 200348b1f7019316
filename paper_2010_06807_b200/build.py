"""Build the sm_100a shared library in-tree (no torch involvement).

    python -m paper_2010_06807_b200.build        # or __graft_entry__.build()

Produces ``paper_2010_06807_b200/libspaqr_b200.so`` with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3``.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libspaqr_b200.so")
SOURCES = ["k_copy.cu", "k_gemm.cu", "k_qr.cu", "k_cpqr.cu", "k_chain.cu", "runtime.cu", "k_krylov.cu",
           "k_wyf.cu", "k_svd.cu"]
# diagnostic host sampling profiler (tools/hostprof.cu): linked in only when
# SPQ_BUILD_HOSTPROF=1, never part of the shipped library
EXTRA = ([os.path.join(os.path.dirname(HERE), "tools", "hostprof.cu")]
         if os.environ.get("SPQ_BUILD_HOSTPROF") == "1" else [])
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-g", "-Xcompiler", "-fno-omit-frame-pointer",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v" if os.environ.get("SPQ_PTXAS_V") else "-O3"]
if os.environ.get("SPQ_PLAIN_SCALARS") == "1":   # A/B: sqrt + divisions in the reflector scalars
    FLAGS.append("-DSPQ_PLAIN_SCALARS")
# diagnostic build: clock64 stamps inside the latency-bound kernels (tools/*_trace.py)
if os.environ.get("SPQ_TRACE") == "1":
    FLAGS.append("-DSPQ_TRACE")
    if os.environ.get("SPQ_TRACE_MMAX"):
        FLAGS.append("-DSPQ_TRACE_MMAX=" + os.environ["SPQ_TRACE_MMAX"])


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "spaqr_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    """Compile every translation unit in parallel, then link the .so."""
    if not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [NVCC, *cflags, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES) + len(EXTRA)) as ex:
        results = list(ex.map(compile_one, SOURCES + EXTRA))
    for obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(obj)}")
        if verbose and (r.stdout or r.stderr):
            sys.stderr.write(r.stdout + r.stderr)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT + ".tmp",
           *[o for o, _ in results], "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libspaqr_b200.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
