"""Proj GEMM + op #4 (+LN2) timing at the bench's shapes (CUDA events, L2 flushed per launch).
usage: python tools/proj_sweep.py [steps]   (SWIN_MLP_DBG2=8 disables the residual L2 prefetch)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(json.dumps(bench.proj_rows(int(sys.argv[1]) if len(sys.argv) > 1 else 20)))
