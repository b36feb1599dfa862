"""Build libsonic.so in-tree with nvcc for sm_100a (explicit gencode; -arch=sm_100a would also
run a generic compute_100 pass that rejects tcgen05)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRCS = ["csrc/sonic_api.cu", "csrc/route.cu", "csrc/aggregate.cu", "csrc/ep.cu", "csrc/peer.cu", "csrc/router.cu", "csrc/fp8.cu"]
DEPS = SRCS + ["csrc/gemm.cuh", "csrc/updown.cuh", "csrc/ptx.cuh", "csrc/sonic_internal.h", "../include/sonic.h"]
OUT = os.path.join(HERE, "libsonic.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xptxas", "-v"]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(os.path.join(HERE, p)) <= t for p in DEPS)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    extra = os.environ.get("SONIC_NVCC_EXTRA", "").split()
    cmd = [NVCC] + FLAGS + extra + ["-o", OUT] + [os.path.join(HERE, s) for s in SRCS]
    r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsonic.so")
    if verbose:
        sys.stderr.write(r.stderr)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
