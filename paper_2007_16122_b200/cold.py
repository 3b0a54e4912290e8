"""Thin ctypes binding over libcold.so (include/cold.h). Argument marshalling only: every
step of the scoring pass runs in the library's CUDA kernels. There is no CPU fallback —
if libcold.so is missing or no sm_100 device is present, the calls raise.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# COLD_LIB_AB: load an A/B variant build instead (tools/ab_build.sh; measurement tooling only)
LIB_PATH = os.environ.get("COLD_LIB_AB") or os.path.join(HERE, "libcold.so")

USER, AD, CROSS = 0, 1, 2
FP32, FP16, BF16 = 0, 1, 2
PRECISION = {"f32": FP32, "f16": FP16, "bf16": BF16}
VALIDATE_IDS = 1

STATUS = {0: "COLD_OK", 1: "COLD_ERR_INVALID_ARG", 2: "COLD_ERR_SHAPE", 3: "COLD_ERR_ID_RANGE",
          4: "COLD_ERR_K_RANGE", 5: "COLD_ERR_NOT_LOADED", 6: "COLD_ERR_PARAMS", 7: "COLD_ERR_OOM",
          8: "COLD_ERR_CUDA", 9: "COLD_ERR_UNSUPPORTED", 10: "COLD_ERR_CAPACITY"}

EXPORTS = ["cold_create", "cold_destroy", "cold_load_params", "cold_score_batch", "cold_score_request",
           "cold_topk", "cold_get_info", "cold_debug_pooled", "cold_debug_features", "cold_debug_rows",
           "cold_status_string", "cold_last_error", "cold_profile", "cold_profile_read", "cold_se_stats",
           "cold_select_groups", "cold_merge_topk", "cold_vps_score", "cold_ctx_clone", "cold_server_create",
           "cold_server_destroy", "cold_server_submit", "cold_server_drain"]
PROF_KINDS = 23
PROF_USER, PROF_GATHER, PROF_TOPK, PROF_FC, PROF_SE_DENSE = 0, 1, 2, 3, 3 + 16
PROF_CHAIN, PROF_TAIL, PROF_MLP_F32 = 20, 21, 22
# cold_config.kernel_flags (include/cold.h COLD_K_*)
K_LAYERWISE, K_NO_U1_MMA, K_SINGLE_CTA, K_PAIR_STREAM, K_STREAM_B = 1, 2, 4, 8, 16
K_TAIL_NONE, K_TAIL3, K_CHAIN_TAIL, K_SERIAL_USER, K_NO_PDL, K_X_ROWS = 32, 64, 128, 256, 512, 1024
K_LAT_TAIL45, K_LAT_FC2_256 = 2048, 4096


class ColdError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class cold_group(C.Structure):
    _fields_ = [("side", C.c_int32), ("pooled", C.c_int32), ("cardinality", C.c_int64),
                ("user_ref", C.c_int32), ("ad_ref", C.c_int32)]


class cold_config(C.Structure):
    _fields_ = [("num_groups", C.c_int32), ("groups", C.POINTER(cold_group)), ("emb_dim", C.c_int32),
                ("num_selected", C.c_int32), ("selected", C.POINTER(C.c_int32)),
                ("num_layers", C.c_int32), ("widths", C.POINTER(C.c_int32)),
                ("activation", C.c_int32), ("linear_log", C.c_int32), ("precision", C.c_int32),
                ("device", C.c_int32), ("max_ads_per_call", C.c_int64), ("max_requests_per_call", C.c_int32),
                ("chunk_ads", C.c_int32), ("flags", C.c_uint32), ("se_mode", C.c_int32),
                ("kernel_flags", C.c_uint32), ("gather_span_chunks", C.c_int32), ("chain_min_ads", C.c_int64),
                ("gather_ring", C.c_int32)]


class cold_params(C.Structure):
    _fields_ = [("table_dtype", C.c_int32), ("tables", C.POINTER(C.c_void_p)),
                ("se_w", C.c_void_p), ("se_b", C.c_void_p),
                ("fc_w", C.POINTER(C.c_void_p)), ("fc_b", C.POINTER(C.c_void_p)),
                ("in_scale", C.c_void_p), ("in_shift", C.c_void_p),
                ("se_w_dense", C.c_void_p), ("se_b_dense", C.c_void_p),
                ("act_slope", C.POINTER(C.c_void_p))]


class cold_server_config(C.Structure):
    _fields_ = [("max_batch_requests", C.c_int32), ("max_batch_ads", C.c_int64), ("top_k", C.c_int32),
                ("max_wait_us", C.c_int32)]


class cold_batch(C.Structure):
    _fields_ = [("num_requests", C.c_int32), ("ad_offsets", C.c_void_p), ("ad_offsets_host", C.c_void_p),
                ("ids", C.POINTER(C.c_void_p)), ("offs", C.POINTER(C.c_void_p)),
                ("offs_host", C.POINTER(C.c_void_p))]


class cold_info(C.Structure):
    _fields_ = [("version", C.c_uint64), ("d_in", C.c_int32), ("d_user", C.c_int32), ("d_ad", C.c_int32),
                ("chunk_ads", C.c_int32), ("kernels_per_chunk", C.c_int32), ("kernels_per_call", C.c_int32),
                ("tensor_core", C.c_int32), ("device_bytes", C.c_int64), ("compressed_activations", C.c_int32),
                ("gather_span_chunks", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Load libcold.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built (python -m paper_2007_16122_b200.build)")
        L = C.CDLL(LIB_PATH)
        L.cold_create.argtypes = [C.POINTER(cold_config), C.POINTER(C.c_void_p)]
        L.cold_destroy.argtypes = [C.c_void_p]
        L.cold_destroy.restype = None
        L.cold_load_params.argtypes = [C.c_void_p, C.POINTER(cold_params), C.POINTER(C.c_uint64)]
        L.cold_score_batch.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_void_p, C.c_void_p]
        L.cold_score_request.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_void_p, C.c_void_p]
        L.cold_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.cold_get_info.argtypes = [C.c_void_p, C.POINTER(cold_info)]
        L.cold_debug_pooled.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_void_p, C.c_void_p]
        L.cold_debug_features.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_void_p, C.c_void_p]
        L.cold_debug_rows.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_int32, C.c_void_p, C.c_int32,
                                      C.c_void_p]
        L.cold_se_stats.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_void_p, C.c_void_p]
        L.cold_select_groups.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.cold_merge_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.cold_vps_score.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.cold_ctx_clone.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.cold_server_create.argtypes = [C.c_void_p, C.POINTER(cold_server_config), C.POINTER(C.c_void_p)]
        L.cold_server_destroy.argtypes = [C.c_void_p]
        L.cold_server_destroy.restype = None
        L.cold_server_submit.argtypes = [C.c_void_p, C.POINTER(cold_batch), C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        L.cold_server_drain.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.cold_profile.argtypes = [C.c_void_p, C.c_int32]
        L.cold_profile_read.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.cold_status_string.restype = C.c_char_p
        L.cold_status_string.argtypes = [C.c_int]
        L.cold_last_error.restype = C.c_char_p
        for f in ["cold_create", "cold_load_params", "cold_score_batch", "cold_score_request", "cold_topk",
                  "cold_get_info", "cold_debug_pooled", "cold_debug_features", "cold_debug_rows",
                  "cold_profile", "cold_profile_read", "cold_se_stats", "cold_select_groups",
                  "cold_merge_topk", "cold_vps_score", "cold_ctx_clone", "cold_server_create",
                  "cold_server_submit", "cold_server_drain"]:
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise ColdError(status, lib().cold_last_error().decode())


def _addr(x) -> int:
    """Address of a torch tensor or numpy array (None -> 0)."""
    if x is None:
        return 0
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def _stream_handle(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Batch:
    """A call's requests (include/cold.h cold_batch). Arrays are torch tensors (device or
    pinned host) or numpy arrays (host). The object keeps them alive."""

    def __init__(self, ad_offsets, ids: Sequence, offs: Sequence, ad_offsets_host: Optional[np.ndarray] = None,
                 offs_host: Optional[Sequence] = None):
        self.ad_offsets = ad_offsets
        self.ids, self.offs = list(ids), list(offs)
        if ad_offsets_host is None:
            ad_offsets_host = ad_offsets.cpu().numpy() if hasattr(ad_offsets, "cpu") else ad_offsets
        self.ad_offsets_host = np.ascontiguousarray(ad_offsets_host, dtype=np.int32)
        M = len(self.ids)
        if offs_host is None:
            offs_host = [None if o is None else (o.cpu().numpy() if hasattr(o, "is_cuda") and o.is_cuda else
                                                 (o.numpy() if hasattr(o, "numpy") and not isinstance(o, np.ndarray) else o))
                         for o in self.offs]
        self.offs_host = [None if o is None else np.ascontiguousarray(o, dtype=np.int32) for o in offs_host]
        self._ids = (C.c_void_p * M)(*[_addr(x) for x in self.ids])
        self._offs = (C.c_void_p * M)(*[_addr(x) for x in self.offs])
        self._offs_host = (C.c_void_p * M)(*[_addr(x) for x in self.offs_host])
        self.R = len(self.ad_offsets_host) - 1
        self.n_ads = int(self.ad_offsets_host[-1])
        self.c = cold_batch(self.R, _addr(self.ad_offsets), self.ad_offsets_host.ctypes.data,
                            C.cast(self._ids, C.POINTER(C.c_void_p)), C.cast(self._offs, C.POINTER(C.c_void_p)),
                            C.cast(self._offs_host, C.POINTER(C.c_void_p)))

    @staticmethod
    def from_numpy(ad_offsets, ids, offs, device="cuda", pin: bool = False):
        """Device batch (pin=False) or pinned-host batch (pin=True) from host numpy arrays."""
        import torch

        def conv(a):
            if a is None:
                return None
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32))
            return t.pin_memory() if pin else t.to(device)
        return Batch(conv(ad_offsets), [conv(x) for x in ids], [conv(x) for x in offs],
                     ad_offsets_host=np.asarray(ad_offsets, np.int32),
                     offs_host=[None if o is None else np.asarray(o, np.int32) for o in offs])


class Context:
    """A cold_ctx: schema, FC widths, precision, capacities."""

    def __init__(self, groups, emb_dim: int, widths: Sequence[int], precision: str = "f16",
                 selected: Optional[Sequence[int]] = None, linear_log: bool = True, device: int = 0,
                 max_ads: int = 1 << 20, max_requests: int = 1024, chunk_ads: int = 0, validate_ids: bool = False,
                 se_mode: str = "group", activation: str = "relu", kernel_flags: int = 0,
                 gather_span_chunks: int = 0, chain_min_ads: int = 0, gather_ring: int = 0):
        """kernel_flags (K_* below), gather_span_chunks, chain_min_ads, gather_ring: kernel-selection
        overrides of include/cold.h (0 = the library's default selection)."""
        L = lib()
        M = len(groups)
        self._groups = (cold_group * M)()
        for i, g in enumerate(groups):
            self._groups[i] = cold_group(int(g.side), int(bool(getattr(g, "pooled", False))), int(g.card),
                                         int(getattr(g, "user_ref", -1)), int(getattr(g, "ad_ref", -1)))
        self._sel = np.asarray(list(selected) if selected else [], np.int32)
        self._widths = np.asarray(list(widths), np.int32)
        cfg = cold_config()
        cfg.num_groups, cfg.groups, cfg.emb_dim = M, self._groups, emb_dim
        cfg.num_selected = len(self._sel)
        cfg.selected = self._sel.ctypes.data_as(C.POINTER(C.c_int32)) if len(self._sel) else None
        cfg.num_layers, cfg.widths = len(self._widths), self._widths.ctypes.data_as(C.POINTER(C.c_int32))
        cfg.activation, cfg.linear_log = {"relu": 0, "prelu": 1}[activation], int(linear_log)
        cfg.precision, cfg.device = PRECISION[precision], device
        cfg.max_ads_per_call, cfg.max_requests_per_call = max_ads, max_requests
        cfg.chunk_ads, cfg.flags = chunk_ads, VALIDATE_IDS if validate_ids else 0
        cfg.se_mode = {"group": 0, "dense": 1}[se_mode]   # AMB-1 readings (include/cold.h)
        cfg.kernel_flags, cfg.gather_span_chunks = int(kernel_flags), int(gather_span_chunks)
        cfg.chain_min_ads, cfg.gather_ring = int(chain_min_ads), int(gather_ring)
        self.precision = precision
        self.device = device
        self.ctx = C.c_void_p()
        _check(L.cold_create(C.byref(cfg), C.byref(self.ctx)))

    def close(self):
        if self.ctx:
            lib().cold_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def clone(self) -> "Context":
        """A context sharing this one's device parameters, with its own workspace (cold_ctx_clone):
        one per concurrent stream. Keep this context alive while the clone is in use."""
        c = Context.__new__(Context)
        c.__dict__.update({k: v for k, v in self.__dict__.items() if k != "ctx"})
        c.ctx = C.c_void_p()
        c._source = self
        _check(lib().cold_ctx_clone(self.ctx, C.byref(c.ctx)))
        return c

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_params(self, tables, se_w, se_b, fc_w, fc_b, table_dtype: str = "f32", in_scale=None,
                    in_shift=None, se_dense=None, act_slope=None) -> int:
        """Host arrays: tables[g] [card, k] (float32, or uint16/float16 bit patterns in the compute
        precision), se_w [M, k], se_b [M], fc_w[l] [out, in], fc_b[l] [out] (float32); optional folded
        input batch norm in_scale / in_shift [D_in] (float32); se_dense = (W [n_sel, D_in], b [n_sel])
        for a se_mode="dense" context; act_slope [L-1] each [out_l] (float32) for activation="prelu"."""
        keep = [np.ascontiguousarray(t) for t in tables]
        sw = np.ascontiguousarray(se_w, np.float32)
        sb = np.ascontiguousarray(se_b, np.float32)
        ws = [np.ascontiguousarray(w, np.float32) for w in fc_w]
        bs = [np.ascontiguousarray(b, np.float32) for b in fc_b]
        tp = (C.c_void_p * len(keep))(*[t.ctypes.data for t in keep])
        wp = (C.c_void_p * len(ws))(*[w.ctypes.data for w in ws])
        bp = (C.c_void_p * len(bs))(*[b.ctypes.data for b in bs])
        isc = None if in_scale is None else np.ascontiguousarray(in_scale, np.float32)
        ish = None if in_shift is None else np.ascontiguousarray(in_shift, np.float32)
        sdw = sdb = None
        if se_dense is not None:
            sdw = np.ascontiguousarray(se_dense[0], np.float32)
            sdb = np.ascontiguousarray(se_dense[1], np.float32)
        sl, slp = None, None
        if act_slope is not None:
            sl = [np.ascontiguousarray(a, np.float32) for a in act_slope]
            slp = (C.c_void_p * len(sl))(*[a.ctypes.data for a in sl])
        p = cold_params(PRECISION[table_dtype], C.cast(tp, C.POINTER(C.c_void_p)), sw.ctypes.data, sb.ctypes.data,
                        C.cast(wp, C.POINTER(C.c_void_p)), C.cast(bp, C.POINTER(C.c_void_p)),
                        None if isc is None else isc.ctypes.data, None if ish is None else ish.ctypes.data,
                        None if sdw is None else sdw.ctypes.data, None if sdb is None else sdb.ctypes.data,
                        None if slp is None else C.cast(slp, C.POINTER(C.c_void_p)))
        v = C.c_uint64()
        _check(lib().cold_load_params(self.ctx, C.byref(p), C.byref(v)))
        return v.value

    def score_batch(self, batch: Batch, scores, stream=None):
        _check(lib().cold_score_batch(self.ctx, C.byref(batch.c), _addr(scores), _stream_handle(stream)))

    def score_request(self, batch: Batch, scores, stream=None):
        _check(lib().cold_score_request(self.ctx, C.byref(batch.c), _addr(scores), _stream_handle(stream)))

    def topk(self, scores, ad_offsets, ad_offsets_host, K: int, idx_out, key_out, bids=None, stream=None):
        aoh = np.ascontiguousarray(ad_offsets_host, np.int32)
        _check(lib().cold_topk(self.ctx, _addr(scores), _addr(ad_offsets), aoh.ctypes.data, len(aoh) - 1, K,
                               _addr(bids), _addr(idx_out), _addr(key_out), _stream_handle(stream)))

    def merge_topk(self, cand_key, cand_idx, G: int, Kl: int, ad_offsets, ad_offsets_host, K: int, idx_out, key_out,
                   stream=None):
        """Merge all-gathered per-rank top-Kl lists [G][R][Kl] into the per-request top-K (F1)."""
        aoh = np.ascontiguousarray(ad_offsets_host, np.int32)
        _check(lib().cold_merge_topk(self.ctx, _addr(cand_key), _addr(cand_idx), G, len(aoh) - 1, Kl,
                                     _addr(ad_offsets), aoh.ctypes.data, K, _addr(idx_out), _addr(key_out),
                                     _stream_handle(stream)))

    def info(self) -> dict:
        i = cold_info()
        _check(lib().cold_get_info(self.ctx, C.byref(i)))
        return {f: getattr(i, f) for f, _ in cold_info._fields_}

    def profile(self, enable: bool):
        _check(lib().cold_profile(self.ctx, int(enable)))

    def profile_read(self, with_flop: bool = False):
        """(total_ms, launches[, algorithmic FLOPs]) per kernel class (PROF_*) since profile(True)."""
        ms = np.zeros(PROF_KINDS, np.float64)
        n = np.zeros(PROF_KINDS, np.int64)
        fl = np.zeros(PROF_KINDS, np.float64)
        _check(lib().cold_profile_read(self.ctx, ms.ctypes.data, n.ctypes.data, fl.ctypes.data))
        return (ms, n, fl) if with_flop else (ms, n)

    def se_stats(self, batch: Batch, stream=None) -> np.ndarray:
        """Mean SE importance weight of every schema group over the batch's ads (cold_se_stats)."""
        out = np.zeros(len(self._groups), np.float64)
        _check(lib().cold_se_stats(self.ctx, C.byref(batch.c), out.ctypes.data, _stream_handle(stream)))
        return out

    def debug_pooled(self, batch: Batch, out, stream=None):
        _check(lib().cold_debug_pooled(self.ctx, C.byref(batch.c), _addr(out), _stream_handle(stream)))

    def debug_features(self, batch: Batch, out, stream=None):
        _check(lib().cold_debug_features(self.ctx, C.byref(batch.c), _addr(out), _stream_handle(stream)))

    def debug_rows(self, batch: Batch, group: int, rows_out, max_rows: int, stream=None):
        _check(lib().cold_debug_rows(self.ctx, C.byref(batch.c), group, _addr(rows_out), max_rows,
                                     _stream_handle(stream)))


def select_groups(mean_s, K: int):
    """The K groups with the largest mean SE weight, ascending schema order (cold_select_groups)."""
    m = np.ascontiguousarray(mean_s, np.float64)
    out = np.empty(K, np.int32)
    _check(lib().cold_select_groups(m.ctypes.data, len(m), K, out.ctypes.data))
    return [int(x) for x in out]


def vps_score(ad_vecs, vec_dtype: str, user_vecs, ad_ids, ad_offsets, ad_offsets_host, scores, stream=None):
    """Vector-product baseline (F4): scores = sigma(v_u[request] . v_a[id]) (cold_vps_score)."""
    aoh = np.ascontiguousarray(ad_offsets_host, np.int32)
    d = int(user_vecs.shape[-1])
    _check(lib().cold_vps_score(_addr(ad_vecs), PRECISION[vec_dtype], int(ad_vecs.shape[0]), d, _addr(user_vecs),
                                _addr(ad_ids), _addr(ad_offsets), aoh.ctypes.data, len(aoh) - 1, _addr(scores),
                                _stream_handle(stream)))


class Server:
    """cold_server: a dispatcher thread that coalesces the requests submitted while the GPU is busy into
    one cold_score_batch + cold_topk call (include/cold.h). Owns the ctx while it lives."""

    def __init__(self, ctx: Context, max_batch_requests: int, max_batch_ads: int, top_k: int, max_wait_us: int = 0):
        cfg = cold_server_config(max_batch_requests, max_batch_ads, top_k, max_wait_us)
        self.srv = C.c_void_p()
        self.top_k = top_k
        self._ctx = ctx
        self._keep = []
        _check(lib().cold_server_create(ctx.ctx, C.byref(cfg), C.byref(self.srv)))

    def submit(self, batch: "Batch", arrival_ns=None):
        """Enqueue the R requests of a host batch (Batch.from_numpy(..., device=None) / pin=True), at
        arrival_ns[r] (CLOCK_MONOTONIC, time.monotonic_ns()) when given. Returns numpy (idx [R, K],
        key [R, K], done_ns [R]) filled asynchronously; valid after drain()."""
        R = len(batch.ad_offsets_host) - 1
        K = self.top_k
        idx = np.zeros((R, K), np.int32)
        key = np.zeros((R, K), np.float32)
        done = np.zeros(R, np.int64)
        arr = None if arrival_ns is None else np.ascontiguousarray(arrival_ns, np.int64)
        self._keep.append((batch, idx, key, done, arr))
        _check(lib().cold_server_submit(self.srv, C.byref(batch.c), None if arr is None else arr.ctypes.data,
                                        idx.ctypes.data, key.ctypes.data, done.ctypes.data))
        return idx, key, done

    def drain(self):
        """Wait for every submitted request; returns (coalesced calls, requests they carried)."""
        b, r = C.c_int64(), C.c_int64()
        _check(lib().cold_server_drain(self.srv, C.byref(b), C.byref(r)))
        self._keep.clear()
        return b.value, r.value

    def close(self):
        if self.srv:
            lib().cold_server_destroy(self.srv)
            self.srv = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
