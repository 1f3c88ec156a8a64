"""Timeline of one CTA of the one-kernel MLP (fused_mlp.cuh trace stamps).
usage: python tools/trace_fused.py <C> <T> [cta]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

C = int(sys.argv[1]) if len(sys.argv) > 1 else 96
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200704
cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L = synth.make_layer(C, 11)
layer = SwinMlpInt8Layer(L, device=0)
print("plan", layer.plan())
x = torch.from_numpy(synth.make_activations(L, T, 12)).cuda()
y = torch.empty((T, C), dtype=torch.int8, device="cuda")
for _ in range(3):
    layer(x, y=y)
buf = torch.zeros(9216, dtype=torch.int64, device="cuda")
layer.set_trace(buf, cta)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
layer(x, y=y)
e.record()
torch.cuda.synchronize()
layer.set_trace(None)
print("kernel ms", s.elapsed_time(e))
t = buf.cpu().numpy().astype(np.int64)
nz = t[t > 0]
t0 = nz.min()
f = lambda v: int(v - t0) if v > 0 else -1
NJ = 4 * C // 128
fc1, fc2 = t[0:512], t[512:1024]
fc1a, fc1b, fc2a, fc2b = t[1024:1536], t[1536:2048], t[6656:7168], t[7168:7680]
fc1w = t[7680:8192]
e5 = t[2048:4096].reshape(1024, 2)
e6 = t[4096:6144].reshape(512, 4)
st = t[6144:8192]
ntile = int((e6[:, 0] > 0).sum())
print(f"NJ={NJ} tiles={ntile}; ns from first stamp")
for i in range(min(ntile, 12)):
    print(f"tile {i}: ep6 start {f(e6[i,0])} pass1 {f(e6[i,2])} stats {f(e6[i,1])} end {f(e6[i,3])} stored {f(st[i])}")
    for j in range(NJ):
        u = i * NJ + j
        print(f"   chunk {u:3d}: FC1 [{f(fc1a[u]):7d},{f(fc1b[u]):7d},w {f(fc1w[u]):7d},{f(fc1[u]):7d}]  ep5 [{f(e5[u,0]):7d},{f(e5[u,1]):7d}]"
              f"  FC2 [{f(fc2a[u]):7d},{f(fc2b[u]):7d},{f(fc2[u]):7d}]")
last = max(f(v) for v in nz)
print("last stamp", last)
cs = t[8192:8192 + 296].reshape(148, 2)
ok = cs[:, 0] > 0
base = cs[ok, 0].min()
st, en = cs[ok, 0] - base, cs[ok, 1] - base
print(f"CTAs {ok.sum()}: entry min {st.min()} max {st.max()} | exit min {en.min()} median {int(np.median(en))} "
      f"max {en.max()} | duration median {int(np.median(en - st))} max {(en - st).max()}")
