"""oracle/mini.py — TEST INFRASTRUCTURE ONLY. Pure-Python fp64 twin of cold_oracle.c.

Written independently of the C file (Python big integers for the hash, math.log /
math.exp, plain lists) for tiny cases (<= a few dozen ads). tests/test_oracle_pins.py
checks the two against each other (P-12) so that a slip in either shows up.
Citations as in cold_oracle.h (P:n = PAPER.md line n).
"""
from __future__ import annotations

import math
import struct

import coldgen

MASK = (1 << 64) - 1


def linear_log(x: float) -> float:
    """P:278-287 Eq. (eq:log), natural log (AMB-4)."""
    if x < -1.0:
        return -math.log(-x) - 1.0
    if x > 1.0:
        return math.log(x) + 1.0
    return x


def sigmoid(z: float) -> float:
    """1/(1+e^-z)."""
    if z >= 0:
        return 1.0 / (1.0 + math.exp(-z))
    e = math.exp(z)
    return e / (1.0 + e)


def fmix64(k: int) -> int:
    k &= MASK
    k ^= k >> 33
    k = (k * 0xff51afd7ed558ccd) & MASK
    k ^= k >> 33
    k = (k * 0xc4ceb9fe1a85ec53) & MASK
    k ^= k >> 33
    return k


def cross_row(g: int, x: int, y: int, card: int) -> int:
    """AMB-9."""
    salt = ((g + 1) * 0x9E3779B97F4A7C15) & MASK
    return (fmix64(fmix64(x ^ salt) ^ y) * card) >> 64


def _value(params: coldgen.Params, g: int, row: int, d: int) -> float:
    t = params.tables[g]
    v = t[row][d]
    if params.table_dtype == "bf16":
        return struct.unpack("<f", struct.pack("<I", int(v) << 16))[0]
    return float(v)


def _bag(schema, batch, g, r, a):
    grp = schema.groups[g]
    if grp.side == coldgen.USER:
        o = batch.offs[g]
        return [int(v) for v in batch.ids[g][o[r]:o[r + 1]]]
    if batch.offs[g] is None:
        return [int(batch.ids[g][a])]
    o = batch.offs[g]
    return [int(v) for v in batch.ids[g][o[a]:o[a + 1]]]


def rows(schema, batch, g, r, a):
    grp = schema.groups[g]
    if grp.side != coldgen.CROSS:
        return _bag(schema, batch, g, r, a)
    xs = _bag(schema, batch, grp.user_ref, r, a)
    ys = _bag(schema, batch, grp.ad_ref, r, a)
    return [cross_row(g, x, y, grp.card) for x in xs for y in ys]


def score_ad(schema, params, batch, r, a, selected=None, linear_log_on=None, prelu=None):
    """p and z for ad a (global index) of request r; every step written out. prelu: per-layer slope
    lists (PReLU hidden activation, x if x > 0 else slope x), else ReLU."""
    sel = list(range(schema.M)) if selected is None else sorted(selected)
    ll = schema.linear_log if linear_log_on is None else linear_log_on
    k = schema.k
    x = []
    for g in sel:
        e = [0.0] * k
        for row in rows(schema, batch, g, r, a):
            for d in range(k):
                e[d] += _value(params, g, row, d)
        if ll:
            e = [linear_log(v) for v in e]
        s = sigmoid(sum(float(params.se_w[g][d]) * e[d] for d in range(k)) + float(params.se_b[g]))
        x.extend(s * v for v in e)
    h = x
    L = len(params.fc_w)
    for l in range(L):
        W, b = params.fc_w[l], params.fc_b[l]
        out = []
        for j in range(W.shape[0]):
            acc = float(b[j])
            for i in range(len(h)):
                acc += float(W[j][i]) * h[i]
            if l == L - 1:
                out.append(acc)
            elif prelu is not None:
                out.append(acc if acc > 0.0 else float(prelu[l][j]) * acc)
            else:
                out.append(max(acc, 0.0))
        h = out
    z = h[1] - h[0] if len(h) == 2 else h[0]
    return sigmoid(z), z


def score(schema, params, batch, selected=None, linear_log_on=None, prelu=None):
    ps, zs = [], []
    for r in range(batch.R):
        for a in range(int(batch.ad_offsets[r]), int(batch.ad_offsets[r + 1])):
            p, z = score_ad(schema, params, batch, r, a, selected, linear_log_on, prelu)
            ps.append(p)
            zs.append(z)
    return ps, zs


def topk(keys, K):
    """P:155; ties by ascending position, NaN last."""
    order = sorted(range(len(keys)), key=lambda i: (math.isnan(keys[i]), -keys[i] if not math.isnan(keys[i]) else 0, i))
    return order[:K]
