"""Seeded synthetic inputs for the COLD scoring pass (shared by tests, smoke and bench).

This module is the ONLY code shared between the CUDA path and the oracle. It
holds none of the method's arithmetic: no pooling, no linear_log, no SE gate,
no FC layer, no cross-feature hash, no top-K. It only describes schemas
(plain data) and draws seeded random numbers (numpy PCG64) for ids, tables,
SE parameters, FC weights and bids. Cross-group ids are never generated: the
method computes them (§3.3 "then computes cross-features").

Schemas (DESIGN.md §3 "input recipe"; SURVEY.md §8 config restatement):
  S-tiny  (BASELINE configs[0]): 8 groups, k=8, FC widths [64, 32, 1], fp32.
  S-paper (configs[1], [2], [4]): 8 user + 8 ad + 8 cross groups, k=16,
          FC 384x1024x512x256x128x64x2 (§4.1), fp16/bf16.
  S-full  (configs[3]): S-paper + 8 more cross groups (M=32, D_in=512).

The paper gives k=16 (L328) and the FC widths (L328) but neither group counts
nor cardinalities; those are readings (DESIGN.md AMB-12).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Union

import numpy as np

USER, AD, CROSS = 0, 1, 2
SIDE_NAMES = {USER: "user", AD: "ad", CROSS: "cross"}


@dataclasses.dataclass(frozen=True)
class Group:
    """One feature group (§3.2: "the embedding of i_th feature group e_i")."""
    name: str
    side: int                  # USER / AD / CROSS
    card: int                  # rows in the group's embedding table
    bag: Optional[tuple] = None  # None = single id; (lo, hi) = bag length range, inclusive
    user_ref: int = -1         # CROSS only: index of the USER group it crosses
    ad_ref: int = -1           # CROSS only: index of the AD group it crosses

    @property
    def pooled(self) -> bool:
        return self.bag is not None


@dataclasses.dataclass(frozen=True)
class Schema:
    name: str
    groups: tuple
    k: int                     # embedding dim (16)
    widths: tuple              # FC widths after D_in, last in {1, 2}
    linear_log: bool = True

    @property
    def M(self) -> int:
        return len(self.groups)

    def side_indices(self, side: int) -> List[int]:
        return [i for i, g in enumerate(self.groups) if g.side == side]


def _cross(name, card, schema_groups, u, a):
    iu = [g.name for g in schema_groups].index(u)
    ia = [g.name for g in schema_groups].index(a)
    return Group(name, CROSS, card, None, iu, ia)


def schema_tiny() -> Schema:
    """S-tiny (BASELINE configs[0]): 3 user, 3 ad, 2 cross groups, k=8, FC [64, 32, 1]."""
    g = [
        Group("user_id", USER, 1000),
        Group("u_cate_bag", USER, 100, (4, 4)),
        Group("u_city", USER, 50),
        Group("ad_id", AD, 1000),
        Group("ad_cate", AD, 100),
        Group("ad_shop", AD, 200),
    ]
    g.append(_cross("u_cate_bag_x_ad_cate", 1024, g, "u_cate_bag", "ad_cate"))
    g.append(_cross("user_id_x_ad_shop", 1024, g, "user_id", "ad_shop"))
    return Schema("S-tiny", tuple(g), 8, (64, 32, 1))


def _paper_groups(extra_cross: bool) -> List[Group]:
    g = [
        Group("user_id", USER, 10**8),
        Group("gender_age", USER, 10**2),
        Group("city", USER, 10**4),
        Group("user_level", USER, 10**2),
        Group("clk_item", USER, 10**7, (32, 32)),
        Group("clk_shop", USER, 10**6, (16, 16)),
        Group("clk_cate", USER, 10**4, (16, 16)),
        Group("clk_brand", USER, 10**5, (16, 16)),
        Group("ad_id", AD, 10**7),
        Group("campaign", AD, 10**6),
        Group("customer", AD, 10**6),
        Group("shop", AD, 10**6),
        Group("brand", AD, 10**5),
        Group("cate", AD, 10**4),
        Group("price_bkt", AD, 10**2),
        Group("ad_type", AD, 10**2),
    ]
    cross = [
        ("clk_cate_x_cate", 10**6, "clk_cate", "cate"),
        ("clk_shop_x_shop", 10**6, "clk_shop", "shop"),
        ("clk_brand_x_brand", 10**6, "clk_brand", "brand"),
        ("user_id_x_cate", 10**7, "user_id", "cate"),
        ("gender_age_x_ad_id", 10**7, "gender_age", "ad_id"),
        ("city_x_shop", 10**6, "city", "shop"),
        ("user_level_x_price_bkt", 10**4, "user_level", "price_bkt"),
        ("gender_age_x_brand", 10**6, "gender_age", "brand"),
    ]
    if extra_cross:
        cross += [
            ("clk_item_x_ad_id", 10**6, "clk_item", "ad_id"),
            ("clk_cate_x_ad_type", 10**4, "clk_cate", "ad_type"),
            ("city_x_cate", 10**6, "city", "cate"),
            ("user_level_x_campaign", 10**6, "user_level", "campaign"),
            ("gender_age_x_price_bkt", 10**4, "gender_age", "price_bkt"),
            ("user_id_x_brand", 10**7, "user_id", "brand"),
            ("clk_brand_x_customer", 10**6, "clk_brand", "customer"),
            ("city_x_ad_type", 10**4, "city", "ad_type"),
        ]
    for name, card, u, a in cross:
        g.append(_cross(name, card, g, u, a))
    return g


PAPER_WIDTHS = (1024, 512, 256, 128, 64, 2)   # PAPER.md L328 §4.1


def schema_paper() -> Schema:
    """S-paper: 8 user + 8 ad + 8 cross groups, k=16, D_in=384 (configs[1],[2],[4])."""
    return Schema("S-paper", tuple(_paper_groups(False)), 16, PAPER_WIDTHS)


def schema_full() -> Schema:
    """S-full: S-paper + 8 cross groups, M=32, D_in=512 (configs[3])."""
    return Schema("S-full", tuple(_paper_groups(True)), 16, PAPER_WIDTHS)


def scaled_schema(schema: Schema, max_card: int) -> Schema:
    """Same structure with every cardinality capped at max_card (small parity cases)."""
    gs = tuple(dataclasses.replace(g, card=min(g.card, max_card)) for g in schema.groups)
    return dataclasses.replace(schema, groups=gs, name=schema.name + f"/cap{max_card}")


# --------------------------------------------------------------------------------------
# storage precision helpers (representation only: RNE rounding of generated values so
# that the stored values both sides see are identical; no method arithmetic)

def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Return float32 values exactly representable in `dtype` ('f32', 'f16', 'bf16'), RNE."""
    x = np.asarray(x, dtype=np.float32)
    if dtype == "f32":
        return x.copy()
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        return bf16_bits_to_f32(f32_to_bf16_bits(x))
    raise ValueError(dtype)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    out = rounded.astype(np.uint16)
    out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


@dataclasses.dataclass
class Params:
    """Model parameters as the caller owns them (host arrays).

    tables[g]: [card, k] in `table_dtype` storage ('f32' -> float32, 'f16' -> float16,
    'bf16' -> uint16 bits). se_w [M, k], se_b [M] float32. fc_w[l] [out, in] float32,
    fc_b[l] [out] float32. When `precision` is f16/bf16, fc_w values are already
    representable in that precision (rounded here, RNE), so every consumer sees the
    same stored weights.
    """
    tables: list
    table_dtype: str
    se_w: np.ndarray
    se_b: np.ndarray
    fc_w: list
    fc_b: list
    precision: str
    init: str
    seed: int

    def table_f64(self, g: int) -> np.ndarray:
        t = self.tables[g]
        if self.table_dtype == "bf16":
            return bf16_bits_to_f32(t).astype(np.float64)
        return t.astype(np.float64)


def _rng(*key) -> np.random.Generator:
    return np.random.default_rng([int(x) & 0xFFFFFFFF for x in key])


def _table(seed: int, g: int, card: int, k: int, amp: float, dtype: str) -> np.ndarray:
    """Uniform [-amp, amp) table, generated in slabs (the 1e8-row user_id table is 6.4 GB in fp32)."""
    out_dtype = {"f32": np.float32, "f16": np.float16, "bf16": np.uint16}[dtype]
    out = np.empty((card, k), dtype=out_dtype)
    slab = max(1, (1 << 24) // k)
    for s, r0 in enumerate(range(0, card, slab)):
        r1 = min(card, r0 + slab)
        v = _rng(seed, 101, g, s).random((r1 - r0, k), dtype=np.float32)
        v = (v - np.float32(0.5)) * np.float32(2.0 * amp)
        if dtype == "f32":
            out[r0:r1] = v
        elif dtype == "f16":
            out[r0:r1] = v.astype(np.float16)
        else:
            out[r0:r1] = f32_to_bf16_bits(v)
    return out


def logit(p: float) -> float:
    return math.log(p / (1.0 - p))


def make_params(schema: Schema, seed: int = 1234, precision: str = "f16",
                init: str = "xavier", se: str = "random", table_amp: float = 0.5,
                table_dtype: Optional[str] = None, d_in: Optional[int] = None,
                base_ctr: float = 0.05) -> Params:
    """Seeded parameters.

    init: 'xavier' (parity init, uniform +-sqrt(6/(fan_in+fan_out))), 'he13' (wide-logit
          stress init, 1.3 * uniform +-sqrt(6/fan_in)), or 'zero' (all FC weights 0).
    se:   'random' (w ~ U(-.25,.25), b ~ U(-1,1)), 'planted' (w = 0, b_g = 3 - 0.5 g),
          'planted_noisy' (w ~ U(-.01,.01), b_g = 3 - 0.5 g), 'identity' (w = 0, b = +40).
    d_in: FC input width (defaults to all groups selected: M * k).
    """
    M, k = schema.M, schema.k
    if table_dtype is None:
        table_dtype = "f32" if precision == "f32" else precision
    tables = [_table(seed, g, grp.card, k, table_amp, table_dtype) for g, grp in enumerate(schema.groups)]
    r = _rng(seed, 202)
    if se == "random":
        se_w = r.uniform(-0.25, 0.25, (M, k)).astype(np.float32)
        se_b = r.uniform(-1.0, 1.0, M).astype(np.float32)
    elif se in ("planted", "planted_noisy"):
        se_w = (np.zeros((M, k)) if se == "planted" else r.uniform(-0.01, 0.01, (M, k))).astype(np.float32)
        se_b = np.array([3.0 - 0.5 * g for g in range(M)], dtype=np.float32)
    elif se == "identity":
        se_w = np.zeros((M, k), np.float32)
        se_b = np.full(M, 40.0, np.float32)
    else:
        raise ValueError(se)
    if d_in is None:
        d_in = M * k
    dims = [d_in] + list(schema.widths)
    fc_w, fc_b = [], []
    for l in range(len(schema.widths)):
        fi, fo = dims[l], dims[l + 1]
        rl = _rng(seed, 303, l)
        if init == "xavier":
            a = math.sqrt(6.0 / (fi + fo))
        elif init == "he13":
            a = 1.3 * math.sqrt(6.0 / fi)
        elif init == "zero":
            a = 0.0
        else:
            raise ValueError(init)
        w = rl.uniform(-a, a, (fo, fi)).astype(np.float32) if a > 0 else np.zeros((fo, fi), np.float32)
        b = rl.uniform(-0.05, 0.05, fo).astype(np.float32)
        if l == len(schema.widths) - 1:
            b = np.zeros(fo, np.float32)
            b[-1] = logit(base_ctr)          # head: p = sigma(z1 - z0) (or sigma(z)) near base_ctr
        fc_w.append(round_to(w, precision))
        fc_b.append(b)
    return Params(tables, table_dtype, se_w, se_b, fc_w, fc_b, precision, init, seed)


def prelu_slopes(schema: Schema, seed: int = 1234, lo: float = 0.05, hi: float = 0.3) -> list:
    """Seeded per-channel PReLU slopes for the hidden layers (the F2 activation variant): [L-1] float32
    arrays of the hidden widths, uniform in [lo, hi)."""
    return [_rng(seed, 404, l).uniform(lo, hi, w).astype(np.float32) for l, w in enumerate(schema.widths[:-1])]


# --------------------------------------------------------------------------------------
# requests

@dataclasses.dataclass
class Batch:
    """R requests, each one user against N_r candidate ads, column-major per group
    (§3.3 "column based"). Per group g:
      USER : offs[g] int32 [R+1] (CSR over requests), ids[g] int32
      AD   : ids[g] int32 [N_tot] (single) or offs[g] [N_tot+1] + ids[g] (bag)
      CROSS: None (computed by the method)
    """
    R: int
    ad_offsets: np.ndarray
    ids: list
    offs: list
    bids: Optional[np.ndarray]
    req_ids: np.ndarray

    @property
    def n_ads(self) -> int:
        return int(self.ad_offsets[-1])


def _draw_ids(rng: np.random.Generator, card: int, n: int, dist: str) -> np.ndarray:
    if dist == "uniform":
        return rng.integers(0, card, n, dtype=np.int64).astype(np.int32)
    if dist == "zipf":   # Zipf(1.05) over [0, card) by continuous inverse CDF
        a = 1.05
        u = rng.random(n)
        x = ((float(card) ** (1 - a) - 1.0) * u + 1.0) ** (1.0 / (1 - a)) - 1.0
        return np.minimum(np.floor(x), card - 1).astype(np.int32)
    raise ValueError(dist)


def make_batch(schema: Schema, req_ids: Union[int, Sequence[int]], n_ads: Union[int, Sequence[int]],
               seed: int = 99, dist: str = "uniform", bids: bool = False) -> Batch:
    """Requests `req_ids` (an int R means range(R)); request r is drawn from its own
    seeded stream, so any subset of a big request stream can be regenerated alone
    (multi-GPU partitions, oracle samples)."""
    if isinstance(req_ids, (int, np.integer)):
        req_ids = range(int(req_ids))
    req_ids = np.asarray(list(req_ids), dtype=np.int64)
    R = len(req_ids)
    if isinstance(n_ads, (int, np.integer)):
        n_list = np.full(R, int(n_ads), dtype=np.int64)
    else:
        n_list = np.asarray(list(n_ads), dtype=np.int64)
        assert len(n_list) == R
    ad_offsets = np.zeros(R + 1, dtype=np.int64)
    np.cumsum(n_list, out=ad_offsets[1:])
    N = int(ad_offsets[-1])
    M = schema.M
    ids = [None] * M
    offs = [None] * M
    # pre-size single-valued ad columns
    for g, grp in enumerate(schema.groups):
        if grp.side == AD and not grp.pooled:
            ids[g] = np.empty(N, dtype=np.int32)
    user_parts = {g: ([], []) for g, grp in enumerate(schema.groups) if grp.side == USER}
    adbag_parts = {g: ([], []) for g, grp in enumerate(schema.groups) if grp.side == AD and grp.pooled}
    bid_arr = np.empty(N, dtype=np.float32) if bids else None
    for i, r in enumerate(req_ids):
        rng = _rng(seed, 404, r)
        a0, a1 = int(ad_offsets[i]), int(ad_offsets[i + 1])
        n = a1 - a0
        for g, grp in enumerate(schema.groups):
            if grp.side == USER:
                L = 1 if not grp.pooled else int(rng.integers(grp.bag[0], grp.bag[1] + 1))
                user_parts[g][0].append(L)
                user_parts[g][1].append(_draw_ids(rng, grp.card, L, dist))
            elif grp.side == AD and not grp.pooled:
                ids[g][a0:a1] = _draw_ids(rng, grp.card, n, dist)
            elif grp.side == AD:
                lens = rng.integers(grp.bag[0], grp.bag[1] + 1, n)
                adbag_parts[g][0].append(lens)
                adbag_parts[g][1].append(_draw_ids(rng, grp.card, int(lens.sum()), dist))
        if bids:
            bid_arr[a0:a1] = rng.uniform(0.1, 10.0, n).astype(np.float32)
    for g, (lens, chunks) in user_parts.items():
        o = np.zeros(R + 1, dtype=np.int64)
        np.cumsum(np.asarray(lens, dtype=np.int64), out=o[1:])
        offs[g] = o.astype(np.int32)
        ids[g] = np.concatenate(chunks).astype(np.int32) if chunks else np.zeros(0, np.int32)
    for g, (lens, chunks) in adbag_parts.items():
        o = np.zeros(N + 1, dtype=np.int64)
        if lens:
            np.cumsum(np.concatenate(lens).astype(np.int64), out=o[1:])
        offs[g] = o.astype(np.int32)
        ids[g] = np.concatenate(chunks).astype(np.int32) if chunks else np.zeros(0, np.int32)
    return Batch(R, ad_offsets.astype(np.int32), ids, offs, bid_arr, req_ids)


def sub_batch(batch: Batch, req_index: Sequence[int]) -> Batch:
    """The requests at positions `req_index` of `batch`, re-packed (host-side slicing)."""
    req_index = list(req_index)
    n_list = [int(batch.ad_offsets[i + 1] - batch.ad_offsets[i]) for i in req_index]
    ad_offsets = np.zeros(len(req_index) + 1, np.int64)
    np.cumsum(n_list, out=ad_offsets[1:])
    ids, offs = [], []
    for g in range(len(batch.ids)):
        if batch.ids[g] is None:
            ids.append(None); offs.append(None); continue
        if batch.offs[g] is not None and len(batch.offs[g]) == batch.R + 1:   # user CSR
            o, v = batch.offs[g], batch.ids[g]
            parts = [v[o[i]:o[i + 1]] for i in req_index]
            no = np.zeros(len(req_index) + 1, np.int64)
            np.cumsum([len(p) for p in parts], out=no[1:])
            ids.append(np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32))
            offs.append(no.astype(np.int32))
        elif batch.offs[g] is None:                                          # ad single
            ids.append(np.concatenate([batch.ids[g][batch.ad_offsets[i]:batch.ad_offsets[i + 1]]
                                       for i in req_index]).astype(np.int32))
            offs.append(None)
        else:                                                                # ad bag
            o, v = batch.offs[g], batch.ids[g]
            lens, parts = [], []
            for i in req_index:
                for a in range(batch.ad_offsets[i], batch.ad_offsets[i + 1]):
                    lens.append(o[a + 1] - o[a]); parts.append(v[o[a]:o[a + 1]])
            no = np.zeros(len(lens) + 1, np.int64)
            np.cumsum(lens, out=no[1:])
            ids.append(np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32))
            offs.append(no.astype(np.int32))
    bids = None
    if batch.bids is not None:
        bids = np.concatenate([batch.bids[batch.ad_offsets[i]:batch.ad_offsets[i + 1]] for i in req_index])
    return Batch(len(req_index), ad_offsets.astype(np.int32), ids, offs, bids,
                 np.asarray([batch.req_ids[i] for i in req_index]))


def selection_all(schema: Schema) -> List[int]:
    return list(range(schema.M))
