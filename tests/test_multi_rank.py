"""Multi-rank host logic on CPU (gloo, world_size 2): the request partition and the top-K gather
give the same per-request top-K as one process scoring the whole stream (oracle scores stand in
for the GPU scorer, which is tested on the GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import coldgen
import oracle
from paper_2007_16122_b200.dist import gather_topk, merge_topk, request_block, split_even

R_PER_RANK, N_ADS, K = 3, 40, 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sch = coldgen.schema_tiny()
    params = coldgen.make_params(sch, seed=3, precision="f32")
    batch = coldgen.make_batch(sch, request_block(R_PER_RANK, rank), N_ADS, seed=4)
    p, _ = oracle.score(oracle.Model(sch, params), batch)
    idx, key = oracle.topk_batch(p, batch.ad_offsets, K)
    gi, gk = gather_topk(torch.from_numpy(idx.reshape(-1).copy()), torch.from_numpy(key.reshape(-1).astype(np.float32)))
    if rank == 0:
        out.put((gi.numpy(), gk.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_and_gather_equal_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    gi, gk = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    # single process over the whole stream
    sch = coldgen.schema_tiny()
    params = coldgen.make_params(sch, seed=3, precision="f32")
    batch = coldgen.make_batch(sch, range(world * R_PER_RANK), N_ADS, seed=4)
    p, _ = oracle.score(oracle.Model(sch, params), batch)
    idx, key = oracle.topk_batch(p, batch.ad_offsets, K)
    np.testing.assert_array_equal(gi.reshape(-1, K), idx)
    np.testing.assert_array_equal(gk.reshape(-1, K), key.astype(np.float32))


def test_split_even_covers_stream():
    for total in (1, 7, 8192):
        for world in (1, 2, 3, 8):
            parts = [split_even(total, world, r) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(total))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_merge_topk_matches_full_sort():
    """F1 merge: per-rank top-K of disjoint ad slices of one request merge to the request's top-K."""
    rng = np.random.default_rng(0)
    for n, G, Kq in [(50, 2, 5), (1000, 4, 100), (37, 3, 37)]:
        keys = np.round(rng.random(n), 2)
        keys[rng.random(n) < 0.05] = np.nan
        want_idx, want_key = oracle.topk(keys, Kq)
        slices = np.array_split(np.arange(n), G)
        kl, pl = [], []
        for sl in slices:
            kk = min(Kq, len(sl))
            i, k = oracle.topk(keys[sl], kk)
            pad = Kq - kk
            kl.append(np.concatenate([k, np.full(pad, np.nan)]))
            pl.append(np.concatenate([sl[i], np.full(pad, 10**9)]))
        mk, mp_ = merge_topk(torch.tensor(np.array(kl)), torch.tensor(np.array(pl)), Kq)
        assert mp_.numpy().tolist() == want_idx.tolist()
