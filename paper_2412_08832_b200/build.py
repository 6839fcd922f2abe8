"""Build the in-tree C-ABI library libhadacore.so for sm_100a (nvcc, no JIT cache).

    python -m paper_2412_08832_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhadacore.so")
SOURCES = [os.path.join(CSRC, "hadacore.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "fwht_kernel.cuh"), os.path.join(CSRC, "fwht_small.cuh"), os.path.join(CSRC, "quant_lab.cuh"), os.path.join(CSRC, "fwht_f32.cuh"), os.path.join(CSRC, "fwht_quant_tc.cuh"), os.path.join(ROOT, "include", "hadacore.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required to build libhadacore.so)")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


# Negative-control library (tests/test_gpu_edge.py): the same source with one sign of the
# H_16 constant flipped (-DHC_NEGCTL); the parity tests must FAIL on it.  Test
# infrastructure only -- the Python binding never loads it.
LIB_NEGCTL = os.path.join(HERE, "libhadacore_negctl.so")
# Timing-perturbation library (tests/test_gpu_jitter.py): -DHC_JITTER inserts random
# nanosleeps at the barrier points of the cluster / warp-specialized kernels; its results
# must be bitwise those of the product library.  Test infrastructure only.
LIB_JITTER = os.path.join(HERE, "libhadacore_jitter.so")


def _cmd(out: str, defines=(), verbose: bool = False):
    return [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
            "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), *defines,
            "-o", out, *SOURCES]


def build(force: bool = False, verbose: bool = False, negctl: bool = True) -> str:
    """Build libhadacore.so (and, with negctl, the negative-control library in parallel)."""
    jobs = []
    if force or needs_build():
        jobs.append((LIB, _cmd(LIB + f".tmp{os.getpid()}", (), verbose)))
    if negctl and (force or not os.path.exists(LIB_NEGCTL) or
                   any(os.path.getmtime(d) > os.path.getmtime(LIB_NEGCTL) for d in DEPS)):
        jobs.append((LIB_NEGCTL, _cmd(LIB_NEGCTL + f".tmp{os.getpid()}", ("-DHC_NEGCTL",), False)))
    if negctl and (force or not os.path.exists(LIB_JITTER) or
                   any(os.path.getmtime(d) > os.path.getmtime(LIB_JITTER) for d in DEPS)):
        jobs.append((LIB_JITTER, _cmd(LIB_JITTER + f".tmp{os.getpid()}", ("-DHC_JITTER",), False)))
    procs = [(dst, cmd[cmd.index("-o") + 1], subprocess.Popen(cmd)) for dst, cmd in jobs]
    for dst, tmp, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc " + os.path.basename(dst))
        os.replace(tmp, dst)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
