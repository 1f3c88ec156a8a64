"""Build an A/B variant of the C-ABI library with extra preprocessor definitions into
build/variants/<name>.so (git-ignored; travels to the GPU box with the snapshot).  Load it with
SWIN_MLP_LIB=build/variants/<name>.so (tools and tests only: bench.py refuses SWIN_MLP_* variables).

usage: python tools/build_variant.py <name> -DFOO=1 [-DBAR=2 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_01169_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.ROOT, "build", "variants")
os.makedirs(out, exist_ok=True)
B.FLAGS = B.FLAGS + defs
B.LIB = os.path.join(out, name + ".so")
if any(d.startswith("-DSWIN_FUSED_REG") for d in defs):   # + the register-path instantiations
    B.UNITS = B.UNITS + [(B.SOURCES[1], [f"-DFUSED_PART={k}"], f"fused_mlp_{k}.o") for k in (4, 5)]
B.UNITS = [(src, extra, f"{name}_{o}") for src, extra, o in B.UNITS]
print(B.build(force=True))
