"""Per-CTA entry/exit (%globaltimer, ns from the first FC1 entry) of both kernels of one MLP
layer run (debug trace buffer), grouped by cluster.  usage: python tools/cta_stamps.py C T [cta]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer, swin_mlp_int8_workspace_bytes

C, T = int(sys.argv[1]), int(sys.argv[2])
cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L = synth.make_layer(C, 11)
layer = SwinMlpInt8Layer(L, device=0)
x = torch.from_numpy(synth.make_activations(L, T, 12)).cuda()
y = torch.empty_like(x)
work = torch.empty(max(swin_mlp_int8_workspace_bytes(layer.handle, T), 128), dtype=torch.uint8, device="cuda")
for _ in range(3):
    layer(x, y=y, workspace=work)
torch.cuda.synchronize()
buf = torch.zeros(9216, dtype=torch.int64, device="cuda")
layer.set_trace(buf, cta)
for _ in range(2):
    buf.zero_()
    layer(x, y=y, workspace=work)
    torch.cuda.synchronize()
layer.set_trace(None)
t = buf.cpu().numpy().astype(np.int64)
print("C", C, "T", T, layer.plan(T))
f1 = t[8192:8192 + 296].reshape(148, 2)
f2 = t[8704:8704 + 296].reshape(148, 2)
base = f1[f1[:, 0] > 0, 0].min()
for name, cs in (("FC1", f1), ("FC2", f2)):
    ok = np.nonzero(cs[:, 0] > 0)[0]
    print(f"== {name}: {ok.size} CTAs")
    rows = [f"{i}:{cs[i,0]-base}-{cs[i,1]-base}" for i in ok]
    for k in range(0, len(rows), 8):
        print("  " + "  ".join(rows[k:k + 8]))
