import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth, oracle
from paper_2402_01169_b200 import SwinMlpInt8Layer
L = synth.make_layer(96, 1096)
T = 1000
X = synth.make_activations(L, T, 5)
layer = SwinMlpInt8Layer(L, device=0)
xd = torch.from_numpy(X).cuda()
zo = torch.empty((T, 96), dtype=torch.float32, device="cuda")
t = layer.run_debug(xd, residual_out=zo)
torch.cuda.synchronize()
m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
Y, yh, z = oracle.ep6(t["acc2"].cpu().numpy(), m2, L.b2, X, L.s_x, L.z_x, L.gamma, L.beta, L.eps, iy, L.z_y)
g = zo.cpu().numpy()
bad = np.argwhere(g != z)
print("n bad", len(bad))
print("cols hist", np.bincount(bad[:, 1], minlength=96))
print("rows first", bad[:10])
r, c = bad[0]
print(g[r, c], z[r, c], X[r, c], t["acc2"][r, c].item())
np.savez("/root/repo/gpurun_out/dbgz.npz", acc2=t["acc2"].cpu().numpy(), X=X, zg=g, zo=z, bad=bad)
