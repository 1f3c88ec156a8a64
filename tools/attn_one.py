"""One attention-half run of a Swin-T b64 stage (for ncu captures): python tools/attn_one.py [stage] [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinAttnInt8Layer, SwinOp1Int8

s = int(sys.argv[1]) if len(sys.argv) > 1 else 0
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
C, S, B = 96 << s, 56 >> s, 64
A = synth.make_attn_layer(C, S, S, 5, M=7, shift=3 if S > 7 else 0)
op1, attn = SwinOp1Int8(A, device=0), SwinAttnInt8Layer(A, device=0)
x = torch.from_numpy(synth.make_block_input(B, S, S, C, 11)).cuda()
for _ in range(iters):
    xw = op1(x)
    a = attn(xw, B)
torch.cuda.synchronize()
print("ok", a.shape)
