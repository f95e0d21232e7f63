"""Build the sm_100a shared library in-tree (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "wb_capi.cu")
LIB = os.path.join(HERE, "libwbflow_b200.so")
# test build of the same sources with every speculative FastDiv unit rejected
# (-DWB_FORCE_REPLAY): all cells, faces and updates take the exact IEEE
# replay path, which tests/test_gpu_replay.py runs against the oracle
LIB_REPLAY = os.path.join(HERE, "libwbflow_b200_replay.so")

# --fmad=false: the reference never contracts a*b+c (Numba/LLVM without
# fastmath); IEEE division/sqrt are nvcc's double-precision defaults and
# --use_fast_math is never used (FP discipline).
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
              "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-Xptxas", "-v"]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d))] + \
        [os.path.join(ROOT, "include", "wbflow_b200.h")]


def needs_build(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force=False, verbose=False, replay=True):
    """Compile the product library and (replay=True) the forced-replay test
    library, both with nvcc for sm_100a, concurrently."""
    nvcc = os.environ.get("NVCC", "nvcc")
    jobs = []
    builds = [(LIB, [])]
    if replay:
        builds.append((LIB_REPLAY, ["-DWB_FORCE_REPLAY"]))
    for lib, extra in builds:
        if not force and not needs_build(lib):
            continue
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", lib, SRC]
        jobs.append((lib, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                           stderr=subprocess.PIPE, text=True)))
    for lib, p in jobs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed building {os.path.basename(lib)}")
        if verbose and lib == LIB:
            sys.stderr.write(err)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
