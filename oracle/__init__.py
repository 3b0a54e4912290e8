"""Oracle — TEST INFRASTRUCTURE ONLY.

A plain fp64 CPU implementation of COLD's scoring pass (oracle/cold_oracle.c) plus
a pure-Python twin for tiny cases (oracle/mini.py). Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package; the
product path (paper_2007_16122_b200/) never does, and shares no code with it.

This module only marshals coldgen objects into the C structs (ctypes) and compiles
the C file with gcc. Every step of the method lives in cold_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

import coldgen

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cold_oracle.c")
LIB = os.path.join(HERE, "libcold_oracle.so")

ORC_OK, ORC_ERR_ARG, ORC_ERR_ID_RANGE, ORC_ERR_K_RANGE = 0, 1, 2, 3
_DT = {"f32": 0, "f16": 1, "bf16": 2}


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, fp64, OpenMP, no FP contraction so the fp32-ordered
    gather mode adds in exactly the written order)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "cold_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", SRC, "-o", LIB + ".tmp", "-lm"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


class _Group(C.Structure):
    _fields_ = [("side", C.c_int32), ("card", C.c_int64), ("user_ref", C.c_int32), ("ad_ref", C.c_int32),
                ("table_dtype", C.c_int32), ("table", C.c_void_p)]


class _Model(C.Structure):
    _fields_ = [("M", C.c_int32), ("k", C.c_int32), ("groups", C.POINTER(_Group)),
                ("n_sel", C.c_int32), ("sel", C.POINTER(C.c_int32)),
                ("se_w", C.POINTER(C.c_double)), ("se_b", C.POINTER(C.c_double)),
                ("se_dense", C.c_int32), ("se_W_dense", C.POINTER(C.c_double)),
                ("se_b_dense", C.POINTER(C.c_double)),
                ("linear_log", C.c_int32), ("ll_after_se", C.c_int32),
                ("L", C.c_int32), ("widths", C.POINTER(C.c_int32)),
                ("W", C.POINTER(C.POINTER(C.c_double))), ("b", C.POINTER(C.POINTER(C.c_double))),
                ("in_scale", C.POINTER(C.c_double)), ("in_shift", C.POINTER(C.c_double)),
                ("activation", C.c_int32), ("slope", C.POINTER(C.POINTER(C.c_double)))]


class _Batch(C.Structure):
    _fields_ = [("R", C.c_int32), ("ad_offsets", C.POINTER(C.c_int32)),
                ("ids", C.POINTER(C.POINTER(C.c_int32))), ("offs", C.POINTER(C.POINTER(C.c_int32)))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.orc_linear_log.restype = C.c_double
        L.orc_linear_log.argtypes = [C.c_double]
        L.orc_sigmoid.restype = C.c_double
        L.orc_sigmoid.argtypes = [C.c_double]
        L.orc_fmix64.restype = C.c_uint64
        L.orc_fmix64.argtypes = [C.c_uint64]
        L.orc_cross_row.restype = C.c_int64
        L.orc_cross_row.argtypes = [C.c_int32, C.c_uint64, C.c_uint64, C.c_int64]
        L.orc_rows.restype = C.c_int64
        L.orc_rows.argtypes = [C.POINTER(_Model), C.POINTER(_Batch), C.c_int32, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_score.restype = C.c_int32
        L.orc_score.argtypes = [C.POINTER(_Model), C.POINTER(_Batch), C.c_void_p, C.c_int64,
                                C.c_void_p, C.c_void_p, C.c_int32]
        L.orc_features.restype = C.c_int32
        L.orc_features.argtypes = [C.POINTER(_Model), C.POINTER(_Batch), C.c_void_p, C.c_int64, C.c_int32,
                                   C.c_void_p]
        L.orc_pooled_f32.restype = C.c_int32
        L.orc_pooled_f32.argtypes = [C.POINTER(_Model), C.POINTER(_Batch), C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_se_gates.restype = C.c_int32
        L.orc_se_gates.argtypes = [C.POINTER(_Model), C.POINTER(_Batch), C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_vps_score.restype = C.c_int32
        L.orc_vps_score.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                    C.c_void_p, C.c_void_p]
        L.orc_topk.restype = C.c_int32
        L.orc_topk.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__({1: "invalid argument", 2: "id out of range", 3: "K out of range"}.get(code, str(code)))
        self.code = code


class Model:
    """Keeps numpy buffers alive for the C struct."""

    def __init__(self, schema: coldgen.Schema, params: coldgen.Params, selected: Optional[Sequence[int]] = None,
                 linear_log: Optional[bool] = None, ll_after_se: bool = False,
                 se_dense: Optional[tuple] = None, in_norm: Optional[tuple] = None,
                 prelu: Optional[Sequence] = None):
        self.schema, self.params = schema, params
        sel = list(range(schema.M)) if selected is None else sorted(selected)
        self._keep = []
        groups = (_Group * schema.M)()
        for i, g in enumerate(schema.groups):
            t = np.ascontiguousarray(params.tables[i])
            self._keep.append(t)
            groups[i] = _Group(g.side, g.card, g.user_ref, g.ad_ref, _DT[params.table_dtype], t.ctypes.data)
        self._groups = groups
        self.sel = np.asarray(sel, np.int32)
        self.se_w = np.ascontiguousarray(params.se_w, np.float64)
        self.se_b = np.ascontiguousarray(params.se_b, np.float64)
        self.widths = np.asarray([w.shape[0] for w in params.fc_w], np.int32)
        self.W = [np.ascontiguousarray(w, np.float64) for w in params.fc_w]
        self.b = [np.ascontiguousarray(b, np.float64) for b in params.fc_b]
        Wp = (C.POINTER(C.c_double) * len(self.W))(*[_ptr(w, C.c_double) for w in self.W])
        bp = (C.POINTER(C.c_double) * len(self.b))(*[_ptr(b, C.c_double) for b in self.b])
        self._Wp, self._bp = Wp, bp
        m = _Model()
        m.M, m.k, m.groups = schema.M, schema.k, groups
        m.n_sel, m.sel = len(sel), _ptr(self.sel, C.c_int32)
        m.se_w, m.se_b = _ptr(self.se_w, C.c_double), _ptr(self.se_b, C.c_double)
        if se_dense is not None:
            self.sWd = np.ascontiguousarray(se_dense[0], np.float64)
            self.sbd = np.ascontiguousarray(se_dense[1], np.float64)
            m.se_dense, m.se_W_dense, m.se_b_dense = 1, _ptr(self.sWd, C.c_double), _ptr(self.sbd, C.c_double)
        m.linear_log = int(schema.linear_log if linear_log is None else linear_log)
        m.ll_after_se = int(ll_after_se)
        m.L, m.widths = len(self.W), _ptr(self.widths, C.c_int32)
        m.W, m.b = C.cast(Wp, C.POINTER(C.POINTER(C.c_double))), C.cast(bp, C.POINTER(C.POINTER(C.c_double)))
        if in_norm is not None:   # (in_scale, in_shift) [n_sel * k]: folded input batch norm
            self.isc = np.ascontiguousarray(in_norm[0], np.float64)
            self.ish = np.ascontiguousarray(in_norm[1], np.float64)
            m.in_scale, m.in_shift = _ptr(self.isc, C.c_double), _ptr(self.ish, C.c_double)
        if prelu is not None:     # PReLU slopes [L-1] each [out_l]
            assert len(prelu) == len(self.W) - 1
            self.slopes = [np.ascontiguousarray(a, np.float64) for a in prelu]
            for a, w in zip(self.slopes, self.W):
                assert a.shape == (w.shape[0],)
            sp = (C.POINTER(C.c_double) * len(self.slopes))(*[_ptr(a, C.c_double) for a in self.slopes])
            self._sp = sp
            m.activation, m.slope = 1, C.cast(sp, C.POINTER(C.POINTER(C.c_double)))
        self.m = m


class BatchView:
    def __init__(self, batch: coldgen.Batch):
        self.batch = batch
        M = len(batch.ids)
        self._keep = []
        ids = (C.POINTER(C.c_int32) * M)()
        offs = (C.POINTER(C.c_int32) * M)()
        for g in range(M):
            if batch.ids[g] is not None:
                a = np.ascontiguousarray(batch.ids[g], np.int32); self._keep.append(a); ids[g] = _ptr(a, C.c_int32)
            if batch.offs[g] is not None:
                a = np.ascontiguousarray(batch.offs[g], np.int32); self._keep.append(a); offs[g] = _ptr(a, C.c_int32)
        self.ad_off = np.ascontiguousarray(batch.ad_offsets, np.int32)
        b = _Batch()
        b.R, b.ad_offsets = batch.R, _ptr(self.ad_off, C.c_int32)
        b.ids = C.cast(ids, C.POINTER(C.POINTER(C.c_int32)))
        b.offs = C.cast(offs, C.POINTER(C.POINTER(C.c_int32)))
        self._ids, self._offs = ids, offs
        self.b = b


def _ads(ad_list):
    if ad_list is None:
        return None, 0
    a = np.ascontiguousarray(ad_list, np.int64)
    return a, len(a)


def score(model: Model, batch: coldgen.Batch, ad_list=None, nthreads: int = 0):
    """Returns (p, z) fp64 for the listed global ads (all when None)."""
    bv = BatchView(batch)
    a, n = _ads(ad_list)
    n_out = batch.n_ads if a is None else n
    p = np.empty(n_out, np.float64)
    z = np.empty(n_out, np.float64)
    rc = lib().orc_score(C.byref(model.m), C.byref(bv.b), None if a is None else a.ctypes.data, n,
                         p.ctypes.data, z.ctypes.data, nthreads)
    if rc:
        raise OracleError(rc)
    return p, z


def features(model: Model, batch: coldgen.Batch, ad_list=None, order: int = 0):
    bv = BatchView(batch)
    a, n = _ads(ad_list)
    n_out = batch.n_ads if a is None else n
    x = np.empty((n_out, len(model.sel) * model.schema.k), np.float64)
    rc = lib().orc_features(C.byref(model.m), C.byref(bv.b), None if a is None else a.ctypes.data, n, order,
                            x.ctypes.data)
    if rc:
        raise OracleError(rc)
    return x


def pooled_f32(model: Model, batch: coldgen.Batch, ad_list=None):
    bv = BatchView(batch)
    a, n = _ads(ad_list)
    n_out = batch.n_ads if a is None else n
    out = np.empty((n_out, len(model.sel), model.schema.k), np.float32)
    rc = lib().orc_pooled_f32(C.byref(model.m), C.byref(bv.b), None if a is None else a.ctypes.data, n,
                              out.ctypes.data)
    if rc:
        raise OracleError(rc)
    return out


def se_gates(model: Model, batch: coldgen.Batch, ad_list=None):
    """s_g of every schema group for the listed ads, [n, M] fp64."""
    bv = BatchView(batch)
    a, n = _ads(ad_list)
    n_out = batch.n_ads if a is None else n
    out = np.empty((n_out, len(model.schema.groups)), np.float64)
    rc = lib().orc_se_gates(C.byref(model.m), C.byref(bv.b), None if a is None else a.ctypes.data, n,
                            out.ctypes.data)
    if rc:
        raise OracleError(rc)
    return out


def vps_score(ad_table, table_dtype: str, user_vecs, ad_offsets, ad_ids):
    """Vector-product model: p[a] = sigma(user_vecs[r] . ad_table[ad_ids[a]]), fp64.
    ad_table holds the stored values (float32, or uint16 bit patterns for 'f16' / 'bf16')."""
    dt = {"f32": 0, "f16": 1, "bf16": 2}[table_dtype]
    tab = np.ascontiguousarray(ad_table, np.float32 if dt == 0 else np.uint16)
    u = np.ascontiguousarray(user_vecs, np.float64)
    ao = np.ascontiguousarray(ad_offsets, np.int32)
    ids = np.ascontiguousarray(ad_ids, np.int32)
    p = np.empty(int(ao[-1]), np.float64)
    rc = lib().orc_vps_score(int(tab.shape[1]), tab.ctypes.data, dt, int(tab.shape[0]), u.ctypes.data, len(ao) - 1,
                             ao.ctypes.data, ids.ctypes.data, p.ctypes.data)
    if rc:
        raise OracleError(rc)
    return p


def select_groups(mean_s, K: int):
    """Feature group selection: rank the groups by importance weight and keep the K with the
    top weights; ties keep schema order (AMB-16). Returned in ascending schema order."""
    mean_s = np.asarray(mean_s, np.float64)
    if not 1 <= K <= len(mean_s):
        raise OracleError(3)
    order = sorted(range(len(mean_s)), key=lambda g: (-mean_s[g], g))
    return sorted(order[:K])


def rows(model: Model, batch: coldgen.Batch, g: int, a: int) -> np.ndarray:
    bv = BatchView(batch)
    n = lib().orc_rows(C.byref(model.m), C.byref(bv.b), g, a, None, 0)
    if n < 0:
        raise OracleError(-n)
    out = np.empty(max(n, 1), np.int64)
    lib().orc_rows(C.byref(model.m), C.byref(bv.b), g, a, out.ctypes.data, n)
    return out[:n]


def topk(key: np.ndarray, K: int):
    key = np.ascontiguousarray(key, np.float64)
    idx = np.empty(K, np.int32)
    kout = np.empty(K, np.float64)
    rc = lib().orc_topk(key.ctypes.data, len(key), K, idx.ctypes.data, kout.ctypes.data)
    if rc:
        raise OracleError(rc)
    return idx, kout


def topk_batch(key: np.ndarray, ad_offsets: np.ndarray, K: int):
    R = len(ad_offsets) - 1
    idx = np.empty((R, K), np.int32)
    kout = np.empty((R, K), np.float64)
    for r in range(R):
        idx[r], kout[r] = topk(key[ad_offsets[r]:ad_offsets[r + 1]], K)
    return idx, kout


def linear_log(x: float) -> float:
    return lib().orc_linear_log(float(x))


def sigmoid(z: float) -> float:
    return lib().orc_sigmoid(float(z))


def fmix64(k: int) -> int:
    return lib().orc_fmix64(k & 0xFFFFFFFFFFFFFFFF)


def cross_row(g: int, x: int, y: int, card: int) -> int:
    return lib().orc_cross_row(g, x, y, card)
