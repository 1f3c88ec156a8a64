"""A/B of the op #6 residual modes (dQ(x) vs fp32 residual, residual_out on/off) for one MLP
layer shape and the proj + op #4 kernel: per-kernel CUDA-event times, L2 flushed per run.
usage: python tools/resid_ab.py C T"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_01169_b200 import SwinMlpInt8Layer, SwinProjInt8Layer  # noqa: E402

C, T = int(sys.argv[1]), int(sys.argv[2])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for k in range(n):
        flush.fill_(k & 0xff)
        ev[k][0].record()
        fn()
        ev[k][1].record()
    torch.cuda.synchronize()
    return round(sorted(a.elapsed_time(b) * 1e3 for a, b in ev)[n // 2], 2)


L = synth.make_layer(C, 77)
h = SwinMlpInt8Layer(L, device=0)
x = torch.from_numpy(synth.make_activations(L, T, 3)).cuda()
r = torch.from_numpy(synth.make_residual(T, C, 4)).cuda()
z = torch.empty_like(r)
y = torch.empty_like(x)
ws = h.workspace(T)
out = {"C": C, "T": T}
out["mlp_dqx"] = timed(lambda: h(x, y=y, workspace=ws))
out["mlp_resid"] = timed(lambda: h(x, residual=r, y=y, workspace=ws))
out["mlp_resid_zout"] = timed(lambda: h(x, residual=r, y=y, residual_out=z, workspace=ws))
out["mlp_dqx_zout"] = timed(lambda: h(x, y=y, residual_out=z, workspace=ws))
P = synth.make_proj(C, 78)
p = SwinProjInt8Layer(P, device=0)
a = torch.from_numpy(synth.make_attn_out(P, T, 5)).cuda()
out["proj_zout"] = timed(lambda: p(a, r, y=y, residual_out=z))
out["proj"] = timed(lambda: p(a, r, y=y))
out["proj_plan"] = p.plan()
print(json.dumps(out))
