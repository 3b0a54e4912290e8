"""Multi-rank host logic on CPU (gloo, world_size 2): the request partition and the top-K gather
give the same per-request top-K as one process scoring the whole stream (oracle scores stand in
for the GPU scorer, which is tested on the GPU)."""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import coldgen
import oracle
from paper_2007_16122_b200.dist import ad_slice, gather_topk, request_block, slice_requests, split_even

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


def _split_worker(rank, world, port, out):
    """F1: every request's ads split across ranks; each rank scores its slices and keeps its top-K;
    the lists are all-gathered rank-major ([G][R][K]) as cold_merge_topk expects."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sch, params, full = _split_case()
    sides = [g.side for g in sch.groups]
    ao, ids, offs, starts = slice_requests(full.ad_offsets, full.ids, full.offs, sides, world, rank)
    mine = dataclasses.replace(full, ad_offsets=ao, ids=ids, offs=offs, bids=None)
    p, _ = oracle.score(oracle.Model(sch, params), mine)
    p = np.round(p, 2)                                    # force ties across ranks
    idx, key = oracle.topk_batch(p, mine.ad_offsets, K)
    gi, gk = gather_topk(torch.from_numpy(idx.reshape(-1).copy()),
                         torch.from_numpy(key.reshape(-1).astype(np.float32)))
    if rank == 0:
        out.put((gi.numpy(), gk.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _split_case():
    sch = coldgen.schema_tiny()
    params = coldgen.make_params(sch, seed=5, precision="f32")
    full = coldgen.make_batch(sch, 3, [40, 57, 33], seed=6)
    return sch, params, full


@pytest.mark.parametrize("world", [2, 3])
def test_split_request_gather_and_merge_rule(world):
    """The host half of F1: slicing (ad_slice rule), scoring per rank, the rank-major all-gather, and
    cold_merge_topk's merge rule (candidates in rank order, top-K by key desc / candidate index,
    position = slice position + floor(g n / G)) reproduce the unsplit per-request top-K."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    gi, gk = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    sch, params, full = _split_case()
    p, _ = oracle.score(oracle.Model(sch, params), full)
    want_idx, want_key = oracle.topk_batch(np.round(p, 2), full.ad_offsets, K)
    G, R = world, full.R
    cand_idx, cand_key = gi.reshape(G, R, K), gk.reshape(G, R, K).astype(np.float64)
    for r in range(R):
        n = int(full.ad_offsets[r + 1] - full.ad_offsets[r])
        keys = np.concatenate([cand_key[g, r] for g in range(G)])
        pos = np.concatenate([cand_idx[g, r] + ad_slice(n, G, g).start for g in range(G)])
        w, _ = oracle.topk(keys, K)
        assert pos[w].tolist() == want_idx[r].tolist()


def test_slice_requests_partition_every_ad():
    sch = coldgen.schema_tiny()
    full = coldgen.make_batch(sch, 4, [5, 1, 17, 9], seed=2)
    sides = [g.side for g in sch.groups]
    for world in (1, 2, 4):
        n_tot = 0
        for rank in range(world):
            ao, ids, offs, starts = slice_requests(full.ad_offsets, full.ids, full.offs, sides, world, rank)
            n_tot += ao[-1]
            for g, gr in enumerate(sch.groups):
                if gr.side == coldgen.AD and offs[g] is None:
                    for r in range(full.R):
                        n = full.ad_offsets[r + 1] - full.ad_offsets[r]
                        sl = ad_slice(int(n), world, rank)
                        np.testing.assert_array_equal(ids[g][ao[r]:ao[r + 1]],
                                                      full.ids[g][full.ad_offsets[r] + sl.start:
                                                                  full.ad_offsets[r] + sl.stop])
        assert n_tot == full.ad_offsets[-1]
