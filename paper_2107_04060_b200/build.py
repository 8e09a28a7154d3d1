"""Build libmg.so (sm_100a) in-tree with nvcc.  No torch extension machinery: the product is a
plain C-ABI shared library (include/mg.h) loaded with ctypes by paper_2107_04060_b200.mg."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmg.so")
SOURCES = ["mg_api.cu", "mg_kernels.cu", "mg_setup.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def regenerate_tables():
    subprocess.check_call([sys.executable, os.path.join(CSRC, "gen_tables.py")], cwd=CSRC,
                          stdout=subprocess.DEVNULL)


def build(verbose: bool = False, force: bool = False) -> str:
    regenerate_tables()
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("mg_tables.h", "mg_internal.h", "mg_kernels.cuh")]
    deps.append(os.path.join(HERE, "..", "include", "mg.h"))
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    extra = os.environ.get("MG_NVCC_EXTRA", "").split()   # diagnostics only (e.g. -DMG_PROL_NOOP)
    cmd = [NVCC, *FLAGS, *extra, "-shared", "-o", LIB, *srcs, "-lcudart"]
    out = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if verbose or out.returncode != 0:
        sys.stderr.write(out.stdout + out.stderr)
    if out.returncode != 0:
        raise RuntimeError("nvcc failed building libmg.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(out.stderr)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
