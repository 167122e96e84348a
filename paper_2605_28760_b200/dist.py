"""Multi-GPU plumbing for the LoZO step, one process per GPU.

Exact-trajectory mode (default): every rank holds a full replica, scores a
contiguous slice of the global minibatch for BOTH probe signs, and the
per-example float64 NLLs are all-gathered (2*B*8 = 256 bytes per step at B=16)
back into the reference's [sign][example] order before the order-defined
canonical mean (numerics.py:271-284), so every rank computes the identical c
and applies the identical rank-r update -- no weight traffic, bitwise-equal
replicas.  The collective is NCCL on GPUs (gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    if B % world:
        raise ValueError(f"global batch {B} does not split over {world} ranks")
    bl = B // world
    return rank * bl, (rank + 1) * bl


def canonical_order(gathered, world: int, bl: int):
    """[rank][sign][b] (all_gather layout) -> [sign][rank*bl + b]."""
    try:
        import torch
        if isinstance(gathered, torch.Tensor):
            return gathered.view(world, 2, bl).transpose(0, 1).reshape(2, world * bl).contiguous()
    except ImportError:
        pass
    return np.asarray(gathered).reshape(world, 2, bl).transpose(1, 0, 2).reshape(2, world * bl)


def exchange_nll(nll_local, world: int, group=None):
    """All-gather the local [2, bl] NLLs and return the global [2, B] tensor."""
    import torch
    import torch.distributed as dist
    bl = nll_local.numel() // 2
    out = torch.empty(world * 2 * bl, dtype=nll_local.dtype, device=nll_local.device)
    dist.all_gather_into_tensor(out, nll_local.reshape(-1).contiguous(), group=group)
    return canonical_order(out, world, bl)
