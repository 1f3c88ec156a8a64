"""Run one layer a few times (ncu target).  usage: python tools/prof_fused.py <C> <T> [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

C = int(sys.argv[1])
T = int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
L = synth.make_layer(C, 11)
layer = SwinMlpInt8Layer(L, device=0)
x = torch.from_numpy(synth.make_activations(L, T, 12)).cuda()
y = torch.empty((T, C), dtype=torch.int8, device="cuda")
for _ in range(iters):
    layer(x, y=y)
torch.cuda.synchronize()
print("ok", C, T, layer.plan())
