"""Host-side cost of enqueueing one layer run (ctypes + validation + maps + launches)."""
import sys, time
import torch
sys.path.insert(0, ".")
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer
for st in range(4):
    L, T, xs = synth.swin_t_batch64_layers()[st]
    layer = SwinMlpInt8Layer(L, device=0)
    x = torch.from_numpy(synth.make_activations(L, T, xs)).cuda()
    y = torch.empty((T, L.C), dtype=torch.int8, device="cuda")
    ws = layer.workspace(T)
    for _ in range(3):
        layer(x, y=y, workspace=ws)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        layer(x, y=y, workspace=ws)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"C={L.C}: enqueue {1e6*(t1-t0)/n:.1f} us/run, wall incl. GPU {1e6*(t2-t0)/n:.1f} us/run")
