"""Multi-GPU plumbing for the token-sharded MLP: one process per
GPU, weights broadcast once from rank 0 (the only collective), tokens split by
whole images, no collective on the hot path.  Backend-agnostic (NCCL on the GPU
box, gloo in the CPU tests); no compute happens here.
"""
from typing import List, Tuple

WEIGHT_FIELDS = ("w1", "s_w1", "b1", "w2", "s_w2", "b2", "gamma", "beta")


def shard_range(n_items: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) share of n_items for `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_tokens(batch: int, tokens_per_image: int, rank: int, world: int) -> Tuple[int, int]:
    """Token rows [t0, t1) of this rank when a batch is split by whole images
    (rows are independent: with the handles' plan hint set to the whole batch's T --
    swin_mlp_int8_set_plan_hint, R20 -- every shard runs the batch's launch plans and
    concat(shards) equals the unsharded run bit for bit; without it a shard small enough to take
    another plan moves Y only inside the R15 tier)."""
    lo, hi = shard_range(batch, rank, world)
    return lo * tokens_per_image, hi * tokens_per_image


def broadcast_layer(layer, device, src: int = 0, group=None) -> List[str]:
    """Replace the layer's weight arrays by tensors broadcast from `src` (one
    collective per array, once at setup).  `layer` fields may be numpy arrays or
    None on every rank; shapes/dtypes must agree (every rank builds the same
    layer description).  Returns the names of the broadcast fields."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    done = []
    for name in WEIGHT_FIELDS:
        a = getattr(layer, name, None)
        if a is None:
            continue
        if isinstance(a, torch.Tensor):
            t = a.to(device).contiguous()
        else:
            a = np.ascontiguousarray(a)
            t = torch.from_numpy(a).to(device) if rank == src else \
                torch.zeros(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=device)
        dist.broadcast(t, src, group=group)
        setattr(layer, name, t)
        done.append(name)
    return done
