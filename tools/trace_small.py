"""Per-CTA timeline of the one-launch small-T plan (small_mlp.cuh): python tools/trace_small.py C T
stamps (ns): 0 start, 1 TMEM, 2 past PDL wait, 3 acc1 ready, 10 acc1 in regs, 11 Hq written, 4 Hq seen by MMA,
5 counted in, 6-8 piece drained, 9 count observed, 14 LN done, 15 exit"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

C, T = int(sys.argv[1]), int(sys.argv[2])
L = synth.make_layer(C, 11)
layer = SwinMlpInt8Layer(L, device=0)
x = torch.from_numpy(synth.make_activations(L, T, 12)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    layer(x, y=y)
torch.cuda.synchronize()
buf = torch.zeros(9216, dtype=torch.int64, device="cuda")
layer.set_trace(buf, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cold in (False, True):
    buf.zero_()
    if cold:
        flush.fill_(1)
    torch.cuda.synchronize()
    layer(x, y=y)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype(np.int64)[: 16 * 148].reshape(148, 16)
    ok = t[:, 0] > 0
    t0 = t[ok, 0].min()
    print("cold" if cold else "hot", "plan", layer.plan(T)["run_plan"], "CTAs", int(ok.sum()))
    for i in np.nonzero(ok)[0][:26]:
        print(i, [int(v - t0) if v else -1 for v in t[i]])
layer.set_trace(None)
