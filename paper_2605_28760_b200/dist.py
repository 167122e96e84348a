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


# ---------------------------------------------------------------- q-direction mode
# SURVEY.md §8(e) mode 2 (zob200.h zo_qdir_*): rank g of G scores reference step
# s = t*G + g -- its own U, window V and minibatch -- on a FULL batch at the shared
# state of macro-step t, so each GPU keeps M = 2*B*T rows (compute-bound) and the
# job processes G reference directions per macro-step ("weak" scaling).  The only
# exchange is the [L+, L-, c, beta] of every rank (32 B); each rank regenerates the
# G counter-keyed U's and applies the G updates in g order -> identical replicas.


def qdir_steps(t: int, world: int) -> list[int]:
    """Reference step indices of macro-step t (rank order)."""
    return [t * world + g for g in range(world)]


def check_qdir(world: int, nu: int, estimator: str = "lozo_lazy") -> None:
    if estimator == "lozo_lazy" and nu % world:
        raise ValueError(f"q-direction mode needs the direction count {world} to divide nu={nu}")


def exchange_out4(out4_local, world: int, group=None):
    """All-gather every rank's [L+, L-, c, beta] -> [world, 4] in rank (= g) order."""
    import torch
    import torch.distributed as dist
    out = torch.empty(world * 4, dtype=out4_local.dtype, device=out4_local.device)
    dist.all_gather_into_tensor(out, out4_local.reshape(-1).contiguous(), group=group)
    return out.view(world, 4)


def fold_due(t: int, world: int, nu: int) -> bool:
    """run_serving_path folds after reference step s when (s+1) % nu == 0
    (runtime.py:327-330); the last step of macro-step t is s = t*world + world - 1."""
    return ((t + 1) * world) % nu == 0
