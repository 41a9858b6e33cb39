"""Build the sm_100a shared library ``lib/libscfa_b200.so`` in-tree with nvcc.

The library is a plain C-ABI ``.so`` (include/scfa_b200.h); the Python host
side loads it with ctypes.  Run ``python -m paper_2306_01160_b200.build``.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libscfa_b200.so")
SOURCES = ["scfa_attn.cu", "scfa_prep.cu", "scfa_sched.cu", "scfa_capi.cu", "scfa_lsh.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc():
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    path = os.path.join(cuda, "bin", "nvcc")
    return path if os.path.exists(path) else "nvcc"


def stale():
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "scfa_b200.h"))
    return any(os.path.getmtime(p) > built for p in deps if os.path.exists(p))


def build(force=False, verbose=False, out=None, extra=()):
    """extra: additional nvcc flags (e.g. -DSCFA_TUNE_* overrides); out: another output path."""
    target = out or LIB_PATH
    if not force and out is None and not stale():
        return LIB_PATH
    os.makedirs(os.path.dirname(target), exist_ok=True)
    tmp = target + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
