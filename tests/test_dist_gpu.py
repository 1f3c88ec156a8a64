"""Two-process token sharding through the CUDA kernels: world size 2 over
gloo, both ranks on cuda:0 (each runs only its own shard; no kernel waits on the other rank).
Rank 0 owns the weights and broadcasts them (the only collective, at setup); every rank creates
its layer from the broadcast bytes, runs its whole-image shard through swin_mlp_int8_run, and
the gathered shards must equal the unsharded single-process run bit for bit.  The handles carry
the plan hint of the whole batch (swin_mlp_int8_set_plan_hint, R20), so the shards
run the batch's launch plans."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    # (C, images, tokens per image): fused C = 96; two-kernel C = 768 (few-tile + split-K shards
    # of one 7x7 window each); C = 384 with several m-tiles per shard
    (96, 6, 49),
    (768, 2, 49),
    (384, 8, 196),
]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    from paper_2402_01169_b200.dist import broadcast_layer, shard_tokens

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    for ci, (C, batch, tpi) in enumerate(CASES):
        # rank 0 holds the real weights; rank 1 starts from other bytes and must receive rank 0's
        L = synth.make_layer(C, 9100 + C if rank == 0 else 9999)
        broadcast_layer(L, torch.device("cpu"))
        csum = int(L.w1.to(torch.int64).sum()) * 3 + int(L.w2.to(torch.int64).sum()) + \
            int(L.s_w1.double().sum() * 1e6) + int(L.gamma.double().sum() * 1e6)
        for n in ("w1", "s_w1", "b1", "w2", "s_w2", "b2", "gamma", "beta"):
            v = getattr(L, n)
            if v is not None:
                setattr(L, n, v.numpy())
        layer = SwinMlpInt8Layer(L, device=0)
        T_full = batch * tpi
        layer.set_plan_hint(T_full)
        Lref = synth.make_layer(C, 9100 + C)
        X = synth.make_activations(Lref, T_full, 31 + ci)
        t0, t1 = shard_tokens(batch, tpi, rank, world)
        x = torch.from_numpy(X[t0:t1]).to(dev)
        y = layer(x).cpu().numpy()
        torch.cuda.synchronize()
        ys, cs = [None] * world, [None] * world
        dist.all_gather_object(ys, y)
        dist.all_gather_object(cs, csum)
        if rank == 0:
            np.save(os.path.join(out_dir, f"y{ci}.npy"), np.concatenate(ys))
            np.save(os.path.join(out_dir, f"c{ci}.npy"), np.array(cs, dtype=np.int64))
        del layer
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_shards_equal_unsharded(tmp_path):
    import torch

    import synth
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for ci, (C, batch, tpi) in enumerate(CASES):
        cs = np.load(tmp_path / f"c{ci}.npy")
        assert cs[0] == cs[1], ("weight checksums differ after the broadcast", C, cs)
        L = synth.make_layer(C, 9100 + C)
        X = synth.make_activations(L, batch * tpi, 31 + ci)
        ref = SwinMlpInt8Layer(L, device=0)(torch.from_numpy(X).cuda()).cpu().numpy()
        y = np.load(tmp_path / f"y{ci}.npy")
        assert y.shape == ref.shape
        np.testing.assert_array_equal(y, ref, err_msg=f"C={C}: concat(shards) != unsharded")
