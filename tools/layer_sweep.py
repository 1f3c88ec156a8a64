"""Per-kernel times of one MLP layer of any shape (FC1+op #5 and FC2+op #6 separately, native
CUDA events on the launching stream, back-to-back runs, L2 flushed before each run) and its plan.
Plan switches are the SWIN_MLP_* environment variables read at create time (see swin_mlp_int8.cu).

usage: python tools/layer_sweep.py C T [iters] [relu|gelu|shiftgelu]   -> one JSON line"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_01169_b200 import SwinMlpInt8Layer, swin_mlp_int8_workspace_bytes  # noqa: E402

C, T = int(sys.argv[1]), int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
act = {"relu": synth.ACT_RELU, "gelu": synth.ACT_GELU, "shiftgelu": synth.ACT_SHIFT_GELU}[sys.argv[4] if len(sys.argv) > 4 else "relu"]
L = synth.make_layer(C, synth.layer_seed(4, 2, 0), act=act)
h = SwinMlpInt8Layer(L, device=0)
x = torch.from_numpy(synth.make_activations(L, T, 7)).cuda()
y = torch.empty_like(x)
work = torch.empty(max(swin_mlp_int8_workspace_bytes(h.handle, T), 128), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    h(x, y=y, workspace=work)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
for k in range(iters):
    flush.fill_(k & 0xff)
    ev[k][0].record()
    h(x, y=y, workspace=work)
    ev[k][1].record()
torch.cuda.synchronize()
us = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
h.profile_begin(iters)
for k in range(iters):
    flush.fill_(k & 0xff)
    h(x, y=y, workspace=work)
torch.cuda.synchronize()
f1, f2, n = h.profile_end()
ops = 2.0 * T * C * 4 * C
env = {k: v for k, v in os.environ.items() if k.startswith("SWIN_MLP_")}
print(json.dumps({"C": C, "T": T, "env": env, "layer_us_median": round(us[len(us) // 2], 2),
                  "fc1_us": round(f1 / max(n, 1) * 1e3, 2), "fc2_us": round(f2 / max(n, 1) * 1e3, 2),
                  "fc1_tops": round(ops / (f1 / max(n, 1) * 1e-3) / 1e12, 1) if f1 else None,
                  "fc2_tops": round(ops / (f2 / max(n, 1) * 1e-3) / 1e12, 1) if f2 else None,
                  "layer_tops": round(2 * ops / (us[len(us) // 2] * 1e-6) / 1e12, 1), "plan": h.plan(T)}), flush=True)
