import sys; sys.path.insert(0, ".")
import torch, numpy as np, synth
from paper_2402_01169_b200 import SwinMlpInt8Layer
L = synth.make_layer(96, 1096)
X = synth.make_activations(L, 300, 5)
layer = SwinMlpInt8Layer(L, device=0)
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
layer.set_trace(buf, 0)
y = layer(torch.from_numpy(X).cuda())
torch.cuda.synchronize()
t = buf.cpu().numpy()
print("markers", hex(t[4095]), hex(t[4094]), hex(t[8191]), "nonzero", np.count_nonzero(t))
print(t[1024:1040], t[2048:2070])
