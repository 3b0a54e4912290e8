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
    order (the global request order under `request_block` / `split_even`; ranks with fewer requests
    pad their blocks, see `unpad_gathered`). NCCL gathers the device tensors in place over
    NVLink; gloo (the CPU tests, and the one-GPU multi-process test) stages device tensors through
    host memory around the same all_gather_into_tensor call."""
    world = dist.get_world_size()
    if out_idx is None:
        out_idx = torch.empty(world * idx.numel(), dtype=idx.dtype, device=idx.device)
        out_key = torch.empty(world * key.numel(), dtype=key.dtype, device=key.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out_idx, idx)
        dist.all_gather_into_tensor(out_key, key)
    else:
        hi, hk = idx.cpu(), key.cpu()
        gi = torch.empty(world * hi.numel(), dtype=hi.dtype)
        gk = torch.empty(world * hk.numel(), dtype=hk.dtype)
        dist.all_gather_into_tensor(gi, hi)
        dist.all_gather_into_tensor(gk, hk)
        out_idx.copy_(gi)
        out_key.copy_(gk)
    return out_idx, out_key


def unpad_gathered(g: "np.ndarray", counts, r_pad: int, K: int):
    """[world * r_pad * K] gathered blocks -> [sum(counts), K]: the first counts[r] requests of
    rank r's block, in rank order."""
    import numpy as np
    g = np.asarray(g).reshape(len(counts), r_pad, K)
    return np.concatenate([g[r, :c] for r, c in enumerate(counts)], axis=0)


def ad_slice(n: int, world: int, rank: int) -> range:
    """F1 split rule (include/cold.h, cold_merge_topk): rank g of G owns ads
    [floor(g n / G), floor((g + 1) n / G)) of a request with n ads."""
    return range(rank * n // world, (rank + 1) * n // world)


def slice_requests(ad_offsets, ids, offs, sides, world: int, rank: int):
    """This rank's share of every request when each request's ads are split across `world` ranks
    (P:248-250 / P:498 split one query's ads into parallel inference calls).
    Columnar arrays in the cold_batch layout (numpy): USER groups keep their per-request bags,
    AD groups keep the ids (single: ids[N]; bag: CSR offs[N+1] rebased) of the rank's ads,
    CROSS groups carry nothing. `sides[g]` is 0 user / 1 ad / 2 cross.
    Returns (ad_offsets, ids, offs, starts) with starts[r] = first ad of the slice in request r."""
    import numpy as np
    ao = np.asarray(ad_offsets, np.int64)
    R = len(ao) - 1
    sel, new_ao, starts = [], [0], []
    for r in range(R):
        sl = ad_slice(int(ao[r + 1] - ao[r]), world, rank)
        sel.append(np.arange(ao[r] + sl.start, ao[r] + sl.stop))
        new_ao.append(new_ao[-1] + len(sl))
        starts.append(sl.start)
    sel = np.concatenate(sel) if sel else np.zeros(0, np.int64)
    out_ids, out_offs = [], []
    for g, side in enumerate(sides):
        if side != 1:
            out_ids.append(ids[g])
            out_offs.append(offs[g])
        elif offs[g] is None:
            out_ids.append(np.ascontiguousarray(np.asarray(ids[g])[sel], np.int32))
            out_offs.append(None)
        else:
            o = np.asarray(offs[g], np.int64)
            lens = o[sel + 1] - o[sel]
            no = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
            idx = np.concatenate([np.arange(o[a], o[a + 1]) for a in sel]) if len(sel) else np.zeros(0, np.int64)
            out_ids.append(np.ascontiguousarray(np.asarray(ids[g])[idx], np.int32))
            out_offs.append(no)
    return np.asarray(new_ao, np.int32), out_ids, out_offs, np.asarray(starts, np.int64)
