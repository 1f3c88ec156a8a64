"""Build the sm_100a C-ABI library in-tree (the .so travels to the GPU box).

nvcc -gencode arch=compute_100a,code=sm_100a: tcgen05.mma.kind::i8 only
assembles for sm_100a (not sm_100f / sm_103a).  -fmad=false: no implicit
contraction — every FMA in the epilogues is an explicit __fmaf_rn, so the
fp32 operation order is exactly the one the oracle defines.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC_DIR = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(SRC_DIR, f) for f in ("swin_mlp_int8.cu", "fused_mlp.cu")]
# (source, extra flags, object) — fused_mlp.cu is compiled once per instantiation part
UNITS = [(SOURCES[0], [], "swin_mlp_int8.o")] + \
    [(SOURCES[1], [f"-DFUSED_PART={k}"], f"fused_mlp_{k}.o") for k in (0, 1, 2, 3)]
DEPS = SOURCES + [os.path.join(SRC_DIR, f) for f in ("mlp_kernels.cuh", "sm100_ptx.cuh", "fused_mlp.cuh", "op5_unfused.cuh",
                                               "attn_kernels.cuh", "small_mlp.cuh")] + \
    [os.path.join(ROOT, "include", f) for f in ("swin_mlp_int8.h", "swin_attn_int8.h")]
LIB = os.path.join(HERE, "libswin_mlp_int8.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
         # a host-only call from device code compiles to UB (the whole kernel folded to EXIT once)
         "-Xcudafe", "--diag_error=20013", "-Xcudafe", "--diag_error=20014", "-Xcudafe", "--diag_error=20015"]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return LIB
    # translation units compile in parallel (the kernel instantiations dominate), then link
    objs, procs = [], []
    for src, extra, oname in UNITS:
        obj = os.path.join(SRC_DIR, oname)
        cmd = [NVCC] + FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", obj, src]
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", LIB] + objs)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
