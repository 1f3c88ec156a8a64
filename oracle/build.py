"""Build the CPU oracle shared library (test infrastructure only).

gcc -O2 -ffp-contract=off -fno-fast-math: every fp32 op rounds where it is
written; the only FMA is the explicit fmaf() the oracle's definition calls for.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRCS = [os.path.join(HERE, f) for f in ("oracle_mlp.c", "oracle_attn.c")]
LIB = os.path.join(HERE, "liboracle_mlp.so")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(f) for f in SRCS):
        return LIB
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fno-builtin-rint",
           "-fopenmp", "-shared", "-fPIC", "-Wall", "-Wextra", "-o", LIB] + SRCS + ["-lm"]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
