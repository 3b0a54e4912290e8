"""Multi-GPU plumbing (torch.distributed): request partitioning and the per-request top-K gather.

Requests are independent ("the pre-rank score of different ads is independent"), so
ranks own disjoint blocks of the request stream and score them with no data-path collective. The
only exchange is the merge of the per-request top-K lists at the end (the paper merges the split
inference queries at the front end, L250): an all-gather of (idx, key) over NCCL on GPUs, over gloo
in the CPU tests.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def request_block(requests_per_rank: int, rank: int) -> range:
    """Weak scaling: rank r owns requests [r * R, (r + 1) * R) of the stream."""
    return range(rank * requests_per_rank, (rank + 1) * requests_per_rank)


def split_even(total: int, world: int, rank: int) -> range:
    """Strong scaling: a fixed total split into near-equal contiguous blocks."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def gather_topk(idx: torch.Tensor, key: torch.Tensor, out_idx: torch.Tensor = None,
                out_key: torch.Tensor = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """All-gather equal-sized per-rank top-K blocks: returns [world * R_local * K] idx / key in rank
    order (the global request order under `request_block`)."""
    world = dist.get_world_size()
    if out_idx is None:
        out_idx = torch.empty(world * idx.numel(), dtype=idx.dtype, device=idx.device)
        out_key = torch.empty(world * key.numel(), dtype=key.dtype, device=key.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out_idx, idx)
        dist.all_gather_into_tensor(out_key, key)
    else:
        dist.all_gather(list(out_idx.chunk(world)), idx)
        dist.all_gather(list(out_key.chunk(world)), key)
    return out_idx, out_key


def merge_topk(keys: torch.Tensor, pos: torch.Tensor, K: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """Merge G partial top-K lists of ONE request (rows of `keys` / `pos`, [G, K'], each sorted by
    (key desc, position asc)) into its top-K, same order, NaN last. Used when one request's ads
    are split across ranks."""
    k = keys.reshape(-1).double()
    p = pos.reshape(-1).long()
    nan = torch.isnan(k)
    # lexicographic (nan, -key, position): sort by position, then stable by key desc, then nan last
    order = torch.argsort(p, stable=True)
    k, p, nan = k[order], p[order], nan[order]
    kk = torch.where(nan, torch.zeros_like(k), -k)
    o2 = torch.argsort(kk, stable=True)
    k, p, nan = k[o2], p[o2], nan[o2]
    o3 = torch.argsort(nan.to(torch.int8), stable=True)
    return k[o3][:K], p[o3][:K]
