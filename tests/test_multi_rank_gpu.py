"""The N > 1 bench path on the one GPU: two processes (gloo; dist.gather_topk stages the device
tensors through host memory around the same all_gather_into_tensor that NCCL runs in place) each
own a libcold context on cuda:0 and run bench.py's own RankStep (configs[4]'s strong-scaling request
partition, cold_score_batch + cold_topk + top-K all-gather, and the e2e form with pinned-host ids and
the D2H of the gathered result) and SplitRequest (F1: one request's ads split across the ranks,
P:248-250). Rank 0 checks the gathered per-request top-K against the fp64 oracle."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R_TOTAL, N_ADS, K = 7, 600, 50


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    import coldgen
    sch = coldgen.scaled_schema(coldgen.schema_paper(), 20000)
    params = coldgen.make_params(sch, seed=81, precision="f16")
    return sch, params


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import bench
    import coldgen
    from paper_2007_16122_b200 import Batch, Context
    from paper_2007_16122_b200.dist import slice_requests

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    sch, params = _case()

    class A:
        scaling, requests = "strong", R_TOTAL
    reqs, r_pad = bench.rank_requests(A, world, rank)
    batch = coldgen.make_batch(sch, reqs, N_ADS, seed=82)
    ctx = Context(sch.groups, sch.k, sch.widths, precision="f16", max_ads=max(batch.n_ads, N_ADS),
                  max_requests=max(batch.R, 1))
    bench.load_ctx_params(ctx, params)
    step = bench.RankStep(ctx, batch, K, world, r_pad, dev)
    step()
    torch.cuda.synchronize()
    gi, gk = (t.cpu().numpy() for t in step.result())
    # e2e form: pinned-host ids, the gathered top-K read back to pinned host memory
    hb = Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs, pin=True)
    step.idx.zero_()
    step.key.zero_()
    step(hb)
    ri, rk = step.result()
    h_idx = torch.empty(ri.numel(), dtype=torch.int32).pin_memory()
    h_key = torch.empty(rk.numel(), dtype=torch.float32).pin_memory()
    h_idx.copy_(ri, non_blocking=True)
    h_key.copy_(rk, non_blocking=True)
    torch.cuda.synchronize()
    # test-only: every rank's scores to rank 0 (the oracle comparison)
    sc = [None] * world
    dist.all_gather_object(sc, (list(reqs), step.scores.cpu().numpy()))
    # F1: two requests, each split across the ranks
    lb = coldgen.make_batch(sch, range(100, 102), N_ADS, seed=83)
    sides = [g.side for g in sch.groups]
    merged, slices = [], []
    for i in range(lb.R):
        one = coldgen.sub_batch(lb, [i])
        ao_s, ids_s, offs_s, _ = slice_requests(one.ad_offsets, one.ids, one.offs, sides, world, rank)
        split = bench.SplitRequest(ctx, N_ADS, int(ao_s[-1]), K, world, dev)
        midx, mkey = split(Batch.from_numpy(ao_s, ids_s, offs_s))
        torch.cuda.synchronize()
        merged.append((midx.cpu().numpy().copy(), mkey.cpu().numpy().copy()))
        slices.append(split.sscores[:int(ao_s[-1])].cpu().numpy().copy())
    sl = [None] * world
    dist.all_gather_object(sl, slices)
    if rank == 0:
        out.put({"gi": gi, "gk": gk, "hi": h_idx.numpy().copy(), "hk": h_key.numpy().copy(), "r_pad": r_pad,
                 "scores": sc, "merged": merged, "slices": sl})
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_bench_rank_step_two_processes_match_oracle():
    import torch.multiprocessing as mp

    import coldgen
    import oracle
    from paper_2007_16122_b200.dist import unpad_gathered

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    sch, params = _case()
    counts = [len(r) for r, _ in res["scores"]]
    assert counts == [4, 3] and sum(counts) == R_TOTAL          # split_even of the 7-request stream
    gi = unpad_gathered(res["gi"], counts, res["r_pad"], K)
    gk = unpad_gathered(res["gk"], counts, res["r_pad"], K)
    # the e2e form (host ids in, D2H of the gathered result) gives the same top-K
    np.testing.assert_array_equal(unpad_gathered(res["hi"], counts, res["r_pad"], K), gi)
    np.testing.assert_array_equal(unpad_gathered(res["hk"], counts, res["r_pad"], K), gk)
    full = coldgen.make_batch(sch, range(R_TOTAL), N_ADS, seed=82)
    p, _ = oracle.score(oracle.Model(sch, params), full)
    got = np.concatenate([s for _, s in res["scores"]]).astype(np.float64)
    assert np.max(np.abs(got - p) / p) <= 2e-2
    # the gathered per-request top-K is exactly the oracle's sort of the GPU scores ...
    oidx, okey = oracle.topk_batch(got, full.ad_offsets, K)
    np.testing.assert_array_equal(gi, oidx)
    np.testing.assert_array_equal(gk.astype(np.float64), okey)
    # ... and agrees with the oracle's own scores' top-K except at ties within the tolerance (P-10)
    ao = full.ad_offsets
    for r in range(R_TOTAL):
        pidx, _ = oracle.topk(p[ao[r]:ao[r + 1]], K)
        kth = np.sort(p[ao[r]:ao[r + 1]])[::-1][K - 1]
        for a in set(pidx.tolist()) ^ set(gi[r].tolist()):
            assert abs(p[ao[r] + a] - kth) <= 2e-2 * kth
    # F1: the merged top-K of each split request equals the oracle's sort of its reassembled scores
    lb = coldgen.make_batch(sch, range(100, 102), N_ADS, seed=83)
    pl, _ = oracle.score(oracle.Model(sch, params), lb)
    for i, (midx, mkey) in enumerate(res["merged"]):
        whole = np.concatenate([res["slices"][g][i] for g in range(world)]).astype(np.float64)
        assert whole.size == N_ADS
        assert np.max(np.abs(whole - pl[i * N_ADS:(i + 1) * N_ADS]) / pl[i * N_ADS:(i + 1) * N_ADS]) <= 2e-2
        widx, wkey = oracle.topk(whole, K)
        np.testing.assert_array_equal(midx, widx)
        np.testing.assert_array_equal(mkey.astype(np.float64), wkey)
