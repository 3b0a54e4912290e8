"""Helpers for the GPU tests: drive libcold through the binding with coldgen inputs."""
import numpy as np

import coldgen


def make_ctx(schema, params, precision=None, selected=None, linear_log=None, max_ads=1 << 16, max_requests=1024,
             chunk_ads=0, validate_ids=False, load=True, **kw):
    from paper_2007_16122_b200 import Context
    precision = precision or params.precision
    ctx = Context(schema.groups, schema.k, schema.widths, precision=precision, selected=selected,
                  linear_log=schema.linear_log if linear_log is None else linear_log,
                  max_ads=max_ads, max_requests=max_requests, chunk_ads=chunk_ads, validate_ids=validate_ids, **kw)
    if load:
        load_params(ctx, params)
    return ctx


def load_params(ctx, params, **kw):
    tables = params.tables
    tdt = params.table_dtype
    if ctx.precision == "f32" and tdt != "f32":          # widen stored 16-bit values (exact)
        tables = [params.table_f64(g).astype(np.float32) for g in range(len(tables))]
        tdt = "f32"
    elif tdt == "f16":
        tables = [t.view(np.uint16) for t in tables]
    return ctx.load_params(tables, params.se_w, params.se_b, params.fc_w, params.fc_b, table_dtype=tdt, **kw)


def device_batch(batch: coldgen.Batch, pin=False):
    from paper_2007_16122_b200 import Batch
    return Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs, pin=pin)


def gpu_scores(ctx, batch: coldgen.Batch, pin=False, host_out=False):
    import torch
    db = device_batch(batch, pin=pin)
    if host_out:
        out = torch.empty(batch.n_ads, dtype=torch.float32).pin_memory()
    else:
        out = torch.empty(batch.n_ads, dtype=torch.float32, device="cuda")
    ctx.score_batch(db, out)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def gpu_topk(ctx, scores_np, ad_offsets, K, bids=None):
    import torch
    s = torch.from_numpy(np.ascontiguousarray(scores_np, np.float32)).cuda()
    ao = torch.from_numpy(np.ascontiguousarray(ad_offsets, np.int32)).cuda()
    R = len(ad_offsets) - 1
    idx = torch.empty(R * K, dtype=torch.int32, device="cuda")
    key = torch.empty(R * K, dtype=torch.float32, device="cuda")
    b = None if bids is None else torch.from_numpy(np.ascontiguousarray(bids, np.float32)).cuda()
    ctx.topk(s, ao, ad_offsets, K, idx, key, bids=b)
    torch.cuda.synchronize()
    return idx.cpu().numpy().reshape(R, K), key.cpu().numpy().reshape(R, K)


def rel_err(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.abs(got - want) / np.maximum(np.abs(want), 1e-30)


def logit(p):
    p = np.clip(np.asarray(p, np.float64), 1e-300, 1 - 1e-16)
    return np.log(p) - np.log1p(-p)
