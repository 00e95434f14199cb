"""In-tree build of the CUDA extension (``libnnp_b200.so``) for sm_100a with nvcc.

The shared library exports exactly the C ABI of ``include/nnp_b200.h``; it links the CUDA
runtime statically and has no Python or torch dependency.
"""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_NAME = "libnnp_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)
SOURCES = ("scan.cu", "nl_kernels.cu", "tn_kernels.cu", "md_kernels.cu", "prior_kernels.cu")
HEADERS = ("nnp_common.cuh", "tn_math.cuh", "tn_gemm.cuh", "tn_gemm_tc5.cuh", os.path.join("..", "..", "include", "nnp_b200.h"))
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
] + [f"-D{d}" for d in os.environ.get("NNP_BUILD_DEFINES", "").split() if d]


def find_nvcc() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        raise RuntimeError("nvcc not found; the CUDA extension cannot be built")
    return nvcc


def is_stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > built for d in deps)


def build_extension(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu for sm_100a and link the shared library next to this file."""
    if not force and not is_stale():
        return LIB_PATH
    nvcc = find_nvcc()
    objs = []
    obj_dir = os.path.join(HERE, "build")
    os.makedirs(obj_dir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [nvcc, "-shared", "-o", LIB_PATH, *objs, "-gencode", "arch=compute_100a,code=sm_100a"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB_PATH


if __name__ == "__main__":
    print(build_extension(force=True, verbose=True))
