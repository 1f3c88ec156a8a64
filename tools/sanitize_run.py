"""One small run of every launch plan (for compute-sanitizer memcheck / racecheck / synccheck):
the one-kernel plan (resident and streamed weights), the two-kernel default, CTA-pair op #6,
few-tile + split-K plans, the unfused (FT-layout) plan, proj + op #4, op #1 and the attention
half.  Checks nothing itself: the sanitizer reports.  usage: python tools/sanitize_run.py"""
import sys

import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinAttnInt8Layer, SwinMlpInt8Layer, SwinOp1Int8, SwinProjInt8Layer

dev = torch.device("cuda:0")
cases = [(96, 300, False), (192, 260, False), (384, 300, False), (512, 1000, False), (768, 49, False),
         (768, 200, False), (1536, 49, False), (384, 300, True)]
for C, T, unf in cases:
    L = synth.make_layer(C, 100 + C)
    layer = SwinMlpInt8Layer(L, device=0, op5_unfused=unf)
    x = torch.from_numpy(synth.make_activations(L, T, 3)).to(dev)
    y = layer(x)
    torch.cuda.synchronize()
    print("mlp", C, T, "unfused" if unf else layer.plan(T).get("run_plan", "fused"), flush=True)
P = synth.make_proj(96, 5)
pl = SwinProjInt8Layer(P, device=0)
a = torch.from_numpy(synth.make_attn_out(P, 300, 5)).to(dev)
r = torch.from_numpy(synth.make_residual(300, 96, 6)).to(dev)
pl(a, r)
torch.cuda.synchronize()
print("proj ok", flush=True)
for C, S, M, sh in ((96, 14, 7, 3), (192, 24, 12, 6)):
    A = synth.make_attn_layer(C, S, S, 7, M=M, shift=sh)
    xb = torch.from_numpy(synth.make_block_input(2, S, S, C, 8)).to(dev)
    xw = SwinOp1Int8(A, device=0)(xb)
    SwinAttnInt8Layer(A, device=0)(xw, 2)
    torch.cuda.synchronize()
    print("attn ok", C, M, flush=True)
