"""Build libqnn.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.environ.get("QNN_LIB_OUT") or os.path.join(PKG, "libqnn.so")
SOURCES = ["abi.cu", "gemm_sm100.cu", "gemm_sm100_split.cu", "gemm_sm100_pair.cu", "gemm_sm100_arows.cu", "gemm_t.cu", "prep.cu", "depthwise.cu", "depthwise_tc.cu", "depthwise_tma.cu", "elementwise.cu", "glue.cu"]
HEADERS = ["common.cuh", "epilogue.cuh", "internal.h", "gemm_sm100.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-cudart", "static",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
# extra defines for profiling builds, e.g. QNN_BUILD_DEFS=-DQNN_GEMM_INSTRUMENT (QNN_GEMM_DEBUG /
# QNN_GEMM_TRACE knobs); rebuild with --force when changing them
FLAGS += os.environ.get("QNN_BUILD_DEFS", "").split()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "qnn.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(PKG, "build" + os.environ.get("QNN_BUILD_TAG", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    errors = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            errors.append(f"--- {src}\n{out.decode()}")
        elif verbose and out:
            print(out.decode(), file=sys.stderr)
    if errors:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errors))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *FLAGS, "-shared", *objs, "-o", tmp])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
