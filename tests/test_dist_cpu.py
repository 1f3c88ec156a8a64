"""Multi-process (world_size 2, gloo, CPU) tests of the token-sharded path's host
logic: weight broadcast from rank 0, sharding by whole images, and
concat(shards) == unsharded (rows are independent; the oracle stands in for the
GPU kernel here, SURVEY §4 "Harness logic without GPUs")."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2402_01169_b200.dist import shard_range, shard_tokens


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1000):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert shard_tokens(64, 3136, 1, 8) == (8 * 3136, 16 * 3136)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2402_01169_b200.dist import broadcast_layer, shard_tokens

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0 owns the real weights; the other ranks start from a different seed
    L = synth.make_layer(96, 777 if rank == 0 else 778)
    names = broadcast_layer(L, torch.device("cpu"))
    assert "w1" in names and "w2" in names
    for n in names:
        setattr(L, n, getattr(L, n).numpy())
    # a batch of 6 "images" of 49 tokens, split by whole images
    batch, tpi = 6, 49
    Lref = synth.make_layer(96, 777)
    X = synth.make_activations(Lref, batch * tpi, 3)
    t0, t1 = shard_tokens(batch, tpi, rank, world)
    y_local = oracle.mlp(L, X[t0:t1])
    sizes = [None] * world
    dist.all_gather_object(sizes, (t0, t1))
    gathered = [None] * world
    dist.all_gather_object(gathered, y_local)
    if rank == 0:
        y = np.concatenate(gathered)
        np.save(os.path.join(out_dir, "sharded.npy"), y)
        np.save(os.path.join(out_dir, "spans.npy"), np.array(sizes))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_broadcast_and_shards_equal_unsharded(tmp_path):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    y = np.load(tmp_path / "sharded.npy")
    spans = np.load(tmp_path / "spans.npy")
    assert spans[0][0] == 0 and spans[-1][1] == 6 * 49
    L = synth.make_layer(96, 777)
    X = synth.make_activations(L, 6 * 49, 3)
    np.testing.assert_array_equal(y, oracle.mlp(L, X))
