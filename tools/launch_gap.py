"""Per-launch time of each Swin-T batch-64 stage layer: back-to-back launches (event pair
around N runs) vs the CTA entry/exit window of one traced run.  Shows how much of a
launch lies outside its CTAs (launch latency, smem reconfiguration, tail).
usage: python tools/launch_gap.py [N]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for L, T, xs in synth.swin_t_batch64_layers():
    lay = SwinMlpInt8Layer(L, device=0)
    x = torch.from_numpy(synth.make_activations(L, T, xs)).cuda()
    y = torch.empty((T, L.C), dtype=torch.int8, device="cuda")
    for _ in range(3):
        lay(x, y=y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(N):
        lay(x, y=y)
    e.record()
    torch.cuda.synchronize()
    per = s.elapsed_time(e) / N * 1e3
    s.record(); lay(x, y=y); e.record(); torch.cuda.synchronize()
    single = s.elapsed_time(e) * 1e3
    buf = torch.zeros(9216, dtype=torch.int64, device="cuda")
    lay.set_trace(buf, 0)
    lay(x, y=y)
    torch.cuda.synchronize()
    lay.set_trace(None)
    t = buf.cpu().numpy().astype(np.int64)
    out = []
    for off in (8192, 8704):
        cs = t[off:off + 296].reshape(148, 2)
        ok = (cs[:, 0] > 0) & (cs[:, 1] > 0)
        if ok.any():
            out.append((int(cs[ok, 1].max() - cs[ok, 0].min()), int(np.median(cs[ok, 1] - cs[ok, 0]))))
    print(f"C={L.C} T={T} plan={lay.plan()} back-to-back {per:.1f} us/launch, single {single:.1f} us, "
          f"CTA window (first entry -> last exit, median CTA) ns {out}")
