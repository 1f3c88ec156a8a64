"""One Swin-T batch-64 step of the FasterTransformer-layout arms (op #5 unfused, NEXT-1),
for ncu launch lists.  usage: python tools/prof_ft.py [gelu|relu] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

act = synth.ACT_GELU if (len(sys.argv) < 2 or sys.argv[1] == "gelu") else synth.ACT_RELU
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
layers = []
for L, T, xs in synth.swin_t_batch64_layers():
    L.act = act
    lay = SwinMlpInt8Layer(L, device=0, op5_unfused=True)
    x = torch.from_numpy(synth.make_activations(L, T, xs)).cuda()
    layers.append((lay, x, torch.empty((T, L.C), dtype=torch.int8, device="cuda")))
for _ in range(reps):
    for lay, x, y in layers:
        lay(x, y=y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for lay, x, y in layers:
    lay(x, y=y)
e.record()
torch.cuda.synchronize()
print("step ms", s.elapsed_time(e))
