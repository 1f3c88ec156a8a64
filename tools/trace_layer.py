"""Pipeline timeline of one CTA (debug trace) for a Swin-T batch-64 stage MLP.
usage: python tools/trace_layer.py <stage | CxT> [cta]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

arg = sys.argv[1] if len(sys.argv) > 1 else "0"
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if "x" in arg:   # "<C>x<T>": any layer shape
    C_, T_ = (int(v) for v in arg.split("x"))
    L, T, xs = synth.make_layer(C_, 11), T_, 12
else:
    L, T, xs = synth.swin_t_batch64_layers()[int(arg)]
layer = SwinMlpInt8Layer(L, device=0)
x = torch.from_numpy(synth.make_activations(L, T, xs)).cuda()
y = torch.empty((T, L.C), dtype=torch.int8, device="cuda")
for _ in range(3):
    layer(x, y=y)
buf = torch.zeros(9216, dtype=torch.int64, device="cuda")
layer.set_trace(buf, cta)
layer(x, y=y)
torch.cuda.synchronize()
layer.set_trace(None)
t = buf.cpu().numpy().astype(np.int64)
print("C", L.C, "T", T, layer.plan())
EPI = ["top", "bufok", "tfull", "pass1", "mean", "var", "-", "end", "sfull", "sread"]
for k, name in ((0, "FC1"), (1, "FC2")):
    base = t[k * 4096:(k + 1) * 4096]
    nz = base[base > 0]
    if nz.size == 0:
        continue
    t0 = nz.min()
    prod = base[0:1024].reshape(512, 2)
    mma4 = base[1024:2048].reshape(256, 4)
    mma = mma4[:, [0, 3]]
    epi = base[2048:3072].reshape(64, 16)
    cst = base[3072:4096].reshape(512, 2)
    print(f"== {name}: ns from first stamp")
    print("tile  prod[s,e]       mma[s,full,issued,e]            const[s,e]      epi: " + " ".join(f"{e:>9s}" for e in EPI))
    n = max(int((mma[:, 0] > 0).sum()), int((epi[:40, 2] > 0).sum()))
    f = lambda v: (v - t0) if v else -1
    for i in range(min(n, 40)):
        ep = " ".join(f"{f(epi[i, j]) if i < 64 else -1:9d}" for j in range(len(EPI)))
        print(f"{i:3d} {f(prod[i,0]):7d},{f(prod[i,1]):7d} {f(mma4[i,0]):7d},{f(mma4[i,1]):7d},{f(mma4[i,2]):7d},{f(mma4[i,3]):7d} "
              f"{f(cst[i,0]):7d},{f(cst[i,1]):7d}  {ep}")
    for i in range(4):
        print("tile", i, "TMA issue", [int(v - t0) if v else -1 for v in epi[40 + i, :6]],
              "MMA full", [int(v - t0) if v else -1 for v in epi[44 + i, :6]])
    rd = [int(v - t0) if v else -1 for v in base[2048 + 16 * 60:2048 + 16 * 62]]
    print("role done per warp", rd[:24], "synced", int(epi[62, 0] - t0) if epi[62, 0] else -1)
    if epi[63, 10]:
        print("store warp done (bulk_wait_all)", epi[63, 10] - t0)
# per-CTA entry / exit (ns, relative to the earliest FC1 entry)
for name, off in (("FC1", 8192), ("FC2", 8704)):
    cs = t[off:off + 2 * 148].reshape(148, 2)
    ok = cs[:, 0] > 0
    if not ok.any():
        continue
    t0c = t[8192:8192 + 296].reshape(148, 2)[:, 0]
    base = t0c[t0c > 0].min()
    st, en = cs[ok, 0] - base, cs[ok, 1] - base
    print(f"{name} CTAs {ok.sum()}: entry min {st.min()} max {st.max()} | exit min {en.min()} "
          f"median {int(np.median(en))} max {en.max()} | duration median {int(np.median(en - st))} max {(en - st).max()}")
