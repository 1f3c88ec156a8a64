"""Run one Swin-T batch-64 stage MLP a few times (for ncu / nsight captures).
usage: python tools/prof_layer.py <stage 0..3 | CxT> [iters] [act relu|gelu] [ln64 0|1]"""
import sys

import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

arg = sys.argv[1] if len(sys.argv) > 1 else "0"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
act = synth.ACT_GELU if len(sys.argv) > 3 and sys.argv[3] == "gelu" else synth.ACT_RELU
ln64 = len(sys.argv) > 4 and sys.argv[4] == "1"
if "x" in arg:   # any layer shape
    C_, T_ = (int(v) for v in arg.split("x"))
    L, T, xs = synth.make_layer(C_, synth.layer_seed(4, 2, 0), act=act), T_, 7
else:
    L, T, xs = synth.swin_t_batch64_layers(act)[int(arg)]
layer = SwinMlpInt8Layer(L, device=0, ln_fp64=ln64)
x = torch.from_numpy(synth.make_activations(L, T, xs)).cuda()
y = torch.empty((T, L.C), dtype=torch.int8, device="cuda")
for _ in range(iters):
    layer(x, y=y)
torch.cuda.synchronize()
print("ok", L.C, T, layer.plan())
