"""Quick GPU diagnostic: run a few layers through run_debug and print how each
tap compares with the oracle (match fractions, first mismatches)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import synth
from paper_2402_01169_b200 import SwinMlpInt8Layer


def cmp(name, got, ref):
    eq = (got == ref)
    frac = eq.mean()
    msg = f"  {name}: match {frac:.6f}"
    if frac < 1:
        idx = np.argwhere(~eq)[:5]
        msg += f" first bad {[(tuple(i), got[tuple(i)], ref[tuple(i)]) for i in idx]}"
        rows_bad = np.unique(np.argwhere(~eq)[:, 0])
        cols_bad = np.unique(np.argwhere(~eq)[:, 1])
        msg += f" rows_bad {len(rows_bad)} cols_bad {len(cols_bad)}"
    print(msg, flush=True)


def main():
    cases = [(96, 200), (192, 130), (384, 129), (768, 64), (1536, 40)]
    if len(sys.argv) > 1:
        cases = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
    dev = torch.device("cuda:0")
    for C, T in cases:
        L = synth.make_layer(C, 1000 + C)
        X = synth.make_activations(L, T, 5)
        t0 = time.time()
        layer = SwinMlpInt8Layer(L, device=0)
        print(f"C={C} T={T} plan={layer.plan()}", flush=True)
        taps = layer.run_debug(torch.from_numpy(X).to(dev))
        torch.cuda.synchronize()
        g = {k: v.cpu().numpy() for k, v in taps.items()}
        print(f"  gpu done {time.time()-t0:.2f}s", flush=True)
        m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
        a1 = oracle.gemm_i8(X, L.w1, L.z_x)
        cmp("acc1", g["acc1"], a1)
        cmp("hidden", g["hidden"], oracle.ep5(g["acc1"], m1, L.b1, ih, L.z_h, act=L.act))
        cmp("acc2", g["acc2"], oracle.gemm_i8(g["hidden"], L.w2, L.z_h))
        Y, yh, z = oracle.ep6(g["acc2"], m2, L.b2, X, L.s_x, L.z_x, L.gamma, L.beta, L.eps, iy, L.z_y)
        cmp("y", g["y"], Y)
        err = np.abs(g["yhat"] - yh).max()
        print(f"  yhat max abs err {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
