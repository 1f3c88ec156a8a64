import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth, oracle
from paper_2402_01169_b200 import SwinMlpInt8Layer
L = synth.make_layer(96, 1096)
X = synth.make_activations(L, 1000, 5)
layer = SwinMlpInt8Layer(L, device=0)
print(layer.plan())
xd = torch.from_numpy(X).cuda()
t = layer.run_debug(xd)
torch.cuda.synchronize()
for k, v in t.items(): print(k, v.abs().float().sum().item())
y = layer(xd); torch.cuda.synchronize()
print("y eq", (y == t["y"]).all().item())
