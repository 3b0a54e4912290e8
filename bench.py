#!/usr/bin/env python
"""bench.py — candidate ads scored/sec (and p99 request latency) of the COLD scoring pass on B200.

Workload (BASELINE.json configs[4], per GPU): a stream of 8192 requests x 10,000 candidate ads,
S-paper schema (8 user + 8 ad + 8 cross groups, k=16, D_in=384), FC 384x1024x512x256x128x64x2,
fp16 storage + fp32 accumulation, linear_log on, SE gate on every group, top-K=500 per request.
One step = score every ad of the rank's requests (cold_score_batch) + per-request top-K
(cold_topk) + NCCL all-gather of the top-K lists (N>1). Requests are partitioned across ranks
(weak scaling: every rank owns its own 8192-request block of the stream). Inputs (2.6 GB of ids +
4.8 GB of tables per GPU) are far larger than L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
  python bench.py --impl reference [--steps K --warmup W]    # the fp64 oracle on the host cores

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import coldgen  # noqa: E402

METRIC = "candidate ads scored/sec and p99 request latency at N ads/request, 1/2/4/8 B200"
PAPER_FLOP_LAYERS = None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="f16", choices=["f16", "bf16", "f32"])
    ap.add_argument("--requests", type=int, default=8192,
                    help="requests per step: the whole stream, partitioned over the GPUs (strong scaling), or "
                         "per GPU with --scaling weak")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--ads", type=int, default=10000, help="ads per request")
    ap.add_argument("--topk", type=int, default=500)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--cap", type=int, default=0, help="cap cardinalities (quick runs only)")
    ap.add_argument("--kernel-flags", type=int, default=0, help="cold_config.kernel_flags (A/B runs)")
    ap.add_argument("--gather-ring", type=int, default=0, help="cold_config.gather_ring (A/B runs)")
    ap.add_argument("--gather-span", type=int, default=0, help="cold_config.gather_span_chunks (A/B runs)")
    ap.add_argument("--chain-min", type=int, default=0, help="cold_config.chain_min_ads (A/B runs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--latency-requests", type=int, default=10000)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--se-sweep", action="store_true",
                    help="BASELINE configs[3]: SE-selected group subsets of S-full, ads/s vs group count")
    ap.add_argument("--se-sample", type=int, default=10000, help="ads in the SE statistics sample (AMB-16)")
    ap.add_argument("--vps", action="store_true",
                    help="F4: the vector-product baseline (P:160-166) on the same request stream, ads/s")
    ap.add_argument("--vps-dim", type=int, default=64)
    ap.add_argument("--se-dense", action="store_true",
                    help="F2: the dense SE reading (AMB-1, P:229-234 Doc B) on the same workload")
    ap.add_argument("--serve", action="store_true",
                    help="serving path: the request-coalescing server (cold_server_*) under open-loop Poisson "
                         "arrivals of configs[1]-shaped requests; p50/p99 end-to-end latency and usable rate")
    ap.add_argument("--serve-requests", type=int, default=6000)
    ap.add_argument("--serve-batch", type=int, default=32, help="max requests coalesced into one call")
    ap.add_argument("--no-serve", action="store_true", help="skip the serving section of the default line")
    ap.add_argument("--latency-sweep", action="store_true",
                    help="SURVEY §8(d) C2: p50/p95/p99 vs N, multi-stream serving (S contexts sharing one "
                         "parameter copy), fp32 / fp16 / bf16 ads/s (the analogue of Table tab:qps_cuda)")
    return ap.parse_args()


def schema_for(args):
    sch = coldgen.schema_paper()
    if args.cap:
        sch = coldgen.scaled_schema(sch, args.cap)
    return sch


def fc_flops_per_ad(sch, d_ac):
    dims = [d_ac] + list(sch.widths)
    return [2 * dims[i] * dims[i + 1] for i in range(len(sch.widths))]


def gather_bytes_per_ad(sch, elem):
    """Algorithmic HBM bytes per ad of the ad+cross gather kernel: gathered rows,
    ad ids, the request index of the ad, and the X_ac write."""
    k = sch.k
    rows, id_bytes = 0, 0
    for g in sch.groups:
        if g.side == coldgen.AD:
            id_bytes += 4
            rows += 1 if not g.pooled else (g.bag[0] + g.bag[1]) / 2
        elif g.side == coldgen.CROSS:
            u = sch.groups[g.user_ref]
            lu = 1 if not u.pooled else (u.bag[0] + u.bag[1]) / 2
            a = sch.groups[g.ad_ref]
            la = 1 if not a.pooled else (a.bag[0] + a.bag[1]) / 2
            rows += lu * la
    n_ac = len([g for g in sch.groups if g.side != coldgen.USER])
    return rows * k * elem + id_bytes + 4 + n_ac * k * elem, rows


# Random-row ceilings measured on this pool's B200s by tools/probes/gather_ceiling.cu
# (profiles/r01/gather_ceiling.jsonl): 32 B rows at uniformly random positions of a table larger than
# L2 come back at 46 G rows/s (1.47 TB/s useful) whatever the number in flight, and ncu counts 125 DRAM
# bytes per such row (the DRAM side moves 128 B per random 32 B sector miss); rows of a 32 MB table
# (L2-resident) come back at 287 G rows/s.
RAND_DRAM_BYTES_PER_ROW = 125.0
RAND_L2_ROWS_PER_S = 287e9
L2_BYTES = 126 * 2**20


def gather_access_model(sch, span_ads, elem, hbm_gbs):
    """Ceiling of the ad + cross gather from the measured random-access rates: each group's rows are
    L2-served when its table fits comfortably in L2 and every row is touched >= 2x per column-wise span,
    else they are random DRAM rows (125 B of DRAM traffic each); L2-class tables still cost one random
    DRAM fetch per row per span. Sequential bytes: ad ids, request index, X_ac write."""
    k = sch.k
    dram_rows = l2_rows = 0.0
    first_touch = 0.0
    for g in sch.groups:
        if g.side == coldgen.USER:
            continue
        if g.side == coldgen.AD:
            rows = 1 if not g.pooled else (g.bag[0] + g.bag[1]) / 2
        else:
            u, a = sch.groups[g.user_ref], sch.groups[g.ad_ref]
            rows = (1 if not u.pooled else (u.bag[0] + u.bag[1]) / 2) * (1 if not a.pooled else (a.bag[0] + a.bag[1]) / 2)
        tbytes = g.card * k * elem
        if tbytes <= L2_BYTES // 3 and span_ads * rows / g.card >= 2:
            l2_rows += rows
            first_touch += min(g.card, span_ads * rows) * RAND_DRAM_BYTES_PER_ROW / span_ads
        else:
            dram_rows += rows
    n_ac = len([g for g in sch.groups if g.side != coldgen.USER])
    seq = 4 * len([g for g in sch.groups if g.side == coldgen.AD]) + 4 + n_ac * k * elem
    dram_b = dram_rows * RAND_DRAM_BYTES_PER_ROW + first_touch + seq
    t_dram = dram_b / (hbm_gbs * 1e9)
    t_l2 = l2_rows / RAND_L2_ROWS_PER_S
    return {"dram_random_rows_per_ad": dram_rows, "l2_rows_per_ad": l2_rows,
            "dram_bytes_per_ad": dram_b, "ceiling_ads_per_s_overlapped": 1.0 / max(t_dram, t_l2),
            "ceiling_ads_per_s_serial": 1.0 / (t_dram + t_l2)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_id), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_ctx_params(ctx, params, se_dense=None):
    tables = params.tables
    tdt = params.table_dtype
    if tdt == "f16":
        tables = [t.view(np.uint16) for t in tables]
    ctx.load_params(tables, params.se_w, params.se_b, params.fc_w, params.fc_b, table_dtype=tdt, se_dense=se_dense)


def dense_se_params(sch, seed):
    """Dense SE gate (AMB-1 Doc B reading): W [M, M k] ~ U(-0.05, 0.05), b [M] ~ U(-1, 1), seeded."""
    rng = np.random.default_rng(seed)
    return (rng.uniform(-0.05, 0.05, (sch.M, sch.M * sch.k)).astype(np.float32),
            rng.uniform(-1, 1, sch.M).astype(np.float32))


# --------------------------------------------------------------------------------------------
def cpu_oracle_sample(sch, params, batch, target_s=15.0, max_ads=None):
    """Time the fp64 oracle (as it stands) on a bounded prefix of request 0's ads."""
    import oracle
    model = oracle.Model(sch, params)
    cores = os.cpu_count() or 1
    oracle.score(model, batch, ad_list=np.arange(min(256, batch.n_ads)), nthreads=cores)   # warm-up
    n0 = min(4096, batch.n_ads)
    t = time.perf_counter()
    oracle.score(model, batch, ad_list=np.arange(n0), nthreads=cores)
    t0 = time.perf_counter() - t
    n = int(min(max_ads or batch.n_ads, max(n0, n0 * target_s / max(t0, 1e-6))))
    t = time.perf_counter()
    oracle.score(model, batch, ad_list=np.arange(n), nthreads=cores)
    dt = time.perf_counter() - t
    return {"value": n / dt, "unit": "ads/s", "cores": cores, "kind": "oracle",
            "sample": f"first {n} ads of the workload's request stream (fp64 C oracle, OpenMP over ads, "
                      f"{dt:.1f} s)"}


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    sch = schema_for(args)
    params = coldgen.make_params(sch, seed=args.seed, precision=args.precision)
    batch = coldgen.make_batch(sch, range(0, 2), args.ads, seed=args.seed + 1)
    model = oracle.Model(sch, params)
    cores = os.cpu_count() or 1
    # size one step to ~3 s of oracle work
    t = time.perf_counter()
    oracle.score(model, batch, ad_list=np.arange(128), nthreads=cores)
    per_ad = (time.perf_counter() - t) / 128
    n = int(min(batch.n_ads, max(128, 3.0 / max(per_ad, 1e-9))))
    ads = np.arange(n)
    for _ in range(args.warmup):
        oracle.score(model, batch, ad_list=ads, nthreads=cores)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.score(model, batch, ad_list=ads, nthreads=cores)
    dt = time.perf_counter() - t
    v = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ads/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(args, sch, args.gpus),
        "cpu_baseline": {"value": v, "unit": "ads/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step = {n} ads of request 0 of the workload stream"},
        "e2e": {"value": v, "unit": "ads/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args, sch, world=1):
    per = "per GPU" if args.scaling == "weak" else f"partitioned over {world} GPU(s)"
    return {"workload": f"BASELINE configs[4]: {args.requests} requests x {args.ads} ads {per} "
                        f"(S-paper schema {sch.name}, M={sch.M}, k={sch.k}, FC {sch.M * sch.k}x"
                        + "x".join(map(str, sch.widths)) + f", {args.precision} + linear_log, top-K={args.topk})",
            "requests": args.requests, "requests_per_gpu": args.requests if args.scaling == "weak"
            else -(-args.requests // world), "ads_per_request": args.ads, "top_k": args.topk,
            "ids": "uniform", "l2": "inputs larger than L2 (ids 2.6 GB + tables 4.8 GB per GPU); no flush",
            "parallelism": f"request partition x{world} ({args.scaling} scaling), replicated params, NCCL top-K "
                           f"all-gather",
            "se": "dense (AMB-1 Doc B reading, user block not hoisted)" if getattr(args, "se_dense", False)
                  else "per-group (AMB-1)"}


# --------------------------------------------------------------------------------------------
def run_se_sweep(args):
    """BASELINE configs[3]: S-full (8 user + 8 ad + 16 cross groups), planted SE
    importance (w ~ U(-.01,.01), b_g = 3 - 0.5 g). The GPU computes mean s_g of every group over a
    10^4-ad sample (cold_se_stats), the top-K_g groups are selected, and each
    lighter model (its own FC1 over D_in = 16 K_g) is timed on 512 requests x 4000 ads + top-500."""
    import torch
    from paper_2007_16122_b200 import Batch, Context, select_groups
    from paper_2007_16122_b200.cold import PROF_GATHER
    torch.cuda.set_device(0)
    sch = coldgen.schema_full()
    R, n_ads, K = 512, 4000, args.topk
    full = coldgen.make_params(sch, seed=args.seed, precision=args.precision, se="planted_noisy")
    sample = coldgen.make_batch(sch, range(2 * 10**7, 2 * 10**7 + max(1, -(-args.se_sample // n_ads))), n_ads,
                                seed=args.seed + 2)
    ctx = Context(sch.groups, sch.k, sch.widths, precision=args.precision, max_ads=sample.n_ads,
                  max_requests=sample.R)
    load_ctx_params(ctx, full)
    mean_s = ctx.se_stats(Batch.from_numpy(sample.ad_offsets, sample.ids, sample.offs))
    ctx.close()
    # the planted gates (b_g = 3 - 0.5 g, |w_g| <= 0.01; coldgen se="planted_noisy") rank the groups in
    # schema order (SURVEY P-11); the oracle parity of cold_se_stats itself is a GPU test
    # (tests/test_gpu_parity.py::test_se_stats_and_selection_match_oracle), not part of the bench
    planted_ok = bool(np.array_equal(np.argsort(-np.asarray(mean_s), kind="stable"), np.arange(sch.M)))
    batch = coldgen.make_batch(sch, range(R), n_ads, seed=args.seed + 1)
    db = Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs)
    dev = torch.device("cuda", 0)
    scores = torch.empty(batch.n_ads, dtype=torch.float32, device=dev)
    idx = torch.empty(R * K, dtype=torch.int32, device=dev)
    key = torch.empty(R * K, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    rows = []
    for kg in (8, 12, 16, 20, 24, 28, 32):
        sel = select_groups(mean_s, kg)
        params = coldgen.make_params(sch, seed=args.seed, precision=args.precision, se="planted_noisy",
                                     d_in=kg * sch.k)
        c = Context(sch.groups, sch.k, sch.widths, precision=args.precision, selected=sel, max_ads=batch.n_ads,
                    max_requests=R)
        load_ctx_params(c, params)

        def step():
            c.score_batch(db, scores)
            c.topk(scores, db.ad_offsets, batch.ad_offsets, K, idx, key)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        c.profile(True)
        for _ in range(args.steps):
            step()
        pm, pn, pf = c.profile_read(with_flop=True)
        c.profile(False)
        info = c.info()
        cls = kernel_classes(sch, pm, pn, pf)
        fc_ms = sum(v["total_ms"] for v in cls.values() if v.get("fc"))
        fc_flop = sum(v.get("flop_per_launch", 0.0) * v["launches"] for v in cls.values() if v.get("fc"))
        n_user = sum(1 for g in sel if sch.groups[g].side == coldgen.USER)
        rows.append({"k_g": kg, "selected_user_ad_cross": [n_user, sum(1 for g in sel if sch.groups[g].side == coldgen.AD),
                                                            sum(1 for g in sel if sch.groups[g].side == coldgen.CROSS)],
                     "d_in": info["d_in"], "d_ad_cross": info["d_ad"], "ads_per_s": batch.n_ads / (ms / 1e3),
                     "ms_per_step": ms, "fc_tflops": fc_flop / (fc_ms / 1e3) / 1e12,
                     "gather_ms": float(pm[PROF_GATHER] / args.steps), "fc_ms": float(fc_ms / args.steps)})
        c.close()
    line = {"metric": METRIC, "value": rows[-1]["ads_per_s"], "unit": "ads/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "dtype": args.precision,
            "data": "synthetic (seeded ids, tables, weights; planted SE importance)",
            "config": {"workload": f"BASELINE configs[3]: S-full (M=32: 8 user + 8 ad + 16 cross), {R} requests x "
                                   f"{n_ads} ads, top-{K}; groups selected by mean SE weight over a "
                                   f"{sample.n_ads}-ad sample (cold_se_stats)"},
            "se_mean_s": [round(float(x), 6) for x in mean_s],
            "se_ranking_matches_planted_order": planted_ok,
            "se_sweep": rows}
    print(json.dumps(line), flush=True)


def run_vps(args):
    """SURVEY §8(f) F4 / Table tab:sys: the vector-product based model served with
    precomputed towers (v_a per ad, v_u per request), p = sigma(v_u . v_a) + per-request top-K, on the
    same request stream shape as the headline run (device-resident inputs, CUDA-event timing)."""
    import torch
    from paper_2007_16122_b200 import Context, vps_score
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    R, n, d, K = args.requests, args.ads, args.vps_dim, args.topk
    card = 10**7                                                    # ad_id cardinality of S-paper
    g = torch.Generator(device=dev).manual_seed(args.seed)
    vecs = ((torch.rand(card, d, device=dev, generator=g) - 0.5) * 0.5).to(torch.float16)
    user = (torch.rand(R, d, device=dev, generator=g) - 0.5) * 0.5
    ids = torch.randint(0, card, (R * n,), device=dev, generator=g, dtype=torch.int32)
    ao = np.arange(0, (R + 1) * n, n, dtype=np.int32)
    d_ao = torch.from_numpy(ao).to(dev)
    scores = torch.empty(R * n, dtype=torch.float32, device=dev)
    idx = torch.empty(R * K, dtype=torch.int32, device=dev)
    key = torch.empty(R * K, dtype=torch.float32, device=dev)
    sch = coldgen.schema_tiny()           # a ctx only for cold_topk's staging; no parameters needed
    ctx = Context(sch.groups, sch.k, sch.widths, precision="f32", max_ads=128, max_requests=R)

    def step():
        vps_score(vecs.view(torch.int16), "f16", user, ids, d_ao, ao, scores)
        ctx.topk(scores, d_ao, ao, K, idx, key)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    e0.record()
    for _ in range(args.steps):
        vps_score(vecs.view(torch.int16), "f16", user, ids, d_ao, ao, scores)
    e1.record()
    e1.synchronize()
    ms_s = e0.elapsed_time(e1) / args.steps
    bytes_per_ad = d * 2 + 4 + 4
    peaks, _ = measured_peaks()
    gbs = R * n * bytes_per_ad / (ms_s / 1e3) / 1e9
    line = {"metric": METRIC, "value": R * n / (ms / 1e3), "unit": "ads/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "dtype": "f16",
            "data": "synthetic (random ad / user tower vectors)",
            "config": {"workload": f"F4 vector-product baseline (P:160-166): {R} requests x {n} ads, d={d}, fp16 "
                                   f"ad vectors for {card} ads, fp32 user vectors, top-{K}"},
            "roofline": {"bound": "hbm", "kernel": "vps", "achieved": gbs, "peak": float(peaks["hbm_gbs"]),
                         "unit": "GB/s", "frac": gbs / float(peaks["hbm_gbs"]),
                         "algorithmic": f"{bytes_per_ad} B/ad (v_a row + id + score)"},
            "score_only_ms": ms_s}
    print(json.dumps(line), flush=True)


def usable_rate(service_ms, limit_ms, seed=7, servers=1):
    """Highest Poisson arrival rate (requests/s) whose simulated open-loop p99 sojourn time stays
    <= limit_ms (the paper's "usable QPS": at most 1% of responses over the limit), for `servers`
    FIFO servers (CUDA streams) whose per-request service times are the measured device times
    `service_ms`. One server: Lindley recursion W_{i+1} = max(0, W_i + S_i - A_{i+1}), sojourn = W + S;
    several: each arrival starts on the earliest-free server. Bisection on the rate."""
    import heapq
    s = np.asarray(service_ms, np.float64)
    gaps = np.random.default_rng(seed).exponential(1.0, size=s.size)   # unit-mean inter-arrival gaps

    def p99(rate):
        a = gaps * (1e3 / rate)   # ms
        out = np.empty_like(s)
        if servers == 1:
            w = 0.0
            for i in range(s.size):
                out[i] = w + s[i]
                if i + 1 < s.size:
                    w = max(0.0, w + s[i] - a[i + 1])
        else:
            free = [0.0] * servers
            t = 0.0
            for i in range(s.size):
                t += a[i]
                start = max(t, heapq.heappop(free))
                heapq.heappush(free, start + s[i])
                out[i] = start + s[i] - t
        return float(np.percentile(out, 99))

    if p99(1.0) > limit_ms:
        return 0.0
    lo, hi = 1.0, 1e3 * servers / float(s.mean())   # stability bound: utilisation < 1
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if p99(mid) <= limit_ms else (lo, mid)
    return lo


def graph_latency(ctx, sch, n, count, K, seed, dist="uniform", dev=None):
    """Per-request latency at N = n over `count` requests, each one a CUDA-graph replay of
    cold_score_request + cold_topk on static device buffers (>= 10^4 sequential
    requests, graph replay). Request i's ids are packed host-side into one int32 row of a device pool;
    the timed region of every request is [one D2D copy of its row into the static buffers (ingest),
    graph replay], bracketed by CUDA events on the replay stream."""
    import torch
    from paper_2007_16122_b200 import Batch
    lb = coldgen.make_batch(sch, range(count), n, seed=seed, dist=dist)
    # static layout: per USER group [L, ids (cap)], per single AD group [n ids]; bags padded to cap
    layout, width = [], 0
    for g, grp in enumerate(sch.groups):
        if grp.side == coldgen.USER:
            cap = 1 if not grp.pooled else grp.bag[1]
            layout.append((g, "user", width, cap))
            width += 2 + cap
        elif grp.side == coldgen.AD:
            if grp.pooled:
                raise ValueError("graph_latency packs single-valued AD groups only")
            layout.append((g, "ad", width, n))
            width += n
    pool = np.zeros((count, width), np.int32)
    for g, kind, off, cap in layout:
        if kind == "user":
            o, v = lb.offs[g], lb.ids[g]
            for i in range(count):
                L = int(o[i + 1] - o[i])
                pool[i, off] = 0
                pool[i, off + 1] = L
                pool[i, off + 2:off + 2 + L] = v[o[i]:o[i + 1]]
        else:
            pool[:, off:off + n] = lb.ids[g].reshape(count, n)
    d_pool = torch.from_numpy(pool).to(dev)
    static = torch.empty(width, dtype=torch.int32, device=dev)
    static.copy_(d_pool[0])
    ids, offs = [None] * sch.M, [None] * sch.M
    for g, kind, off, cap in layout:
        if kind == "user":
            offs[g] = static[off:off + 2]
            ids[g] = static[off + 2:off + 2 + cap]
        else:
            ids[g] = static[off:off + n]
    ao = np.asarray([0, n], np.int32)
    d_ao = torch.from_numpy(ao).to(dev)
    sb = Batch(d_ao, ids, offs, ad_offsets_host=ao,
               offs_host=[None if o is None else np.asarray([0, 1], np.int32) for o in offs])
    kk = min(K, n)
    sc = torch.empty(n, dtype=torch.float32, device=dev)
    idx = torch.empty(kk, dtype=torch.int32, device=dev)
    key = torch.empty(kk, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):   # warm-up outside capture: sizes the library's lazily grown buffers
            ctx.score_request(sb, sc, stream=s)
            ctx.topk(sc, d_ao, ao, kk, idx, key, stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        ctx.score_request(sb, sc, stream=s)
        ctx.topk(sc, d_ao, ao, kk, idx, key, stream=s)
    # parity of the replay against a direct call on request 1
    with torch.cuda.stream(s):
        static.copy_(d_pool[1])
        graph.replay()
        g_idx = idx.clone()
        ctx.score_request(sb, sc, stream=s)
        ctx.topk(sc, d_ao, ao, kk, idx, key, stream=s)
    s.synchronize()
    replay_ok = bool(torch.equal(g_idx, idx))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(count)]
    with torch.cuda.stream(s):
        for i in range(min(20, count)):
            static.copy_(d_pool[i])
            graph.replay()
        for i in range(count):
            evs[i][0].record(s)
            static.copy_(d_pool[i])
            graph.replay()
            evs[i][1].record(s)
    s.synchronize()
    lat = np.array([a.elapsed_time(b) for a, b in evs])
    del graph
    return {"n_ads": n, "top_k": kk, "requests": count, "ids": dist, "p50_ms": float(np.percentile(lat, 50)),
            "p95_ms": float(np.percentile(lat, 95)), "p99_ms": float(np.percentile(lat, 99)),
            "mean_ms": float(lat.mean()), "ads_per_s": n / (float(lat.mean()) / 1e3),
            "usable_rps_p99_le_1ms": usable_rate(lat, 1.0), "usable_rps_p99_le_10ms": usable_rate(lat, 10.0),
            "replay_matches_direct_call": replay_ok,
            "timing": "CUDA-graph replay of score_request + top-K per request (ingest = one D2D copy of the "
                      "request's packed ids, inside the timed region), device events, one stream; usable_rps: "
                      "Lindley-recursion open-loop Poisson arrivals over these measured service times (P:442 rule)"}


def serve_rates(srv, hb, n_ads, rates, seed=11):
    """Open-loop Poisson arrivals at each offered rate (requests/s): the C-side submit enqueues request i
    at its arrival time; latency = completion (dispatcher publishes the top-K to host memory) - arrival,
    host CLOCK_MONOTONIC. Returns one row per rate."""
    rows = []
    R = len(hb.ad_offsets_host) - 1
    for lam in rates:
        gaps = np.random.default_rng(seed).exponential(1e9 / lam, R)
        arrival = (time.monotonic_ns() + 5_000_000 + np.cumsum(gaps)).astype(np.int64)
        _, _, done = srv.submit(hb, arrival_ns=arrival)
        calls, reqs = srv.drain()
        lat = (done - arrival) / 1e6
        span = (done.max() - arrival.min()) / 1e9
        rows.append({"offered_rps": float(lam), "offered_ads_per_s": float(lam * n_ads),
                     "achieved_ads_per_s": float(R * n_ads / span), "p50_ms": float(np.percentile(lat, 50)),
                     "p99_ms": float(np.percentile(lat, 99)), "mean_ms": float(lat.mean()),
                     "failed": int((done < 0).sum())})
    return rows


def serve_sweep(ctx, sch, args, n_requests, B, fractions=(0.1, 0.25, 0.5, 0.7, 0.85, 0.95)):
    """The coalescing server on `ctx` (which it owns until it returns): closed-loop capacity, then open-loop
    Poisson arrivals at fractions of it; usable rate at p99 <= 1 ms / 10 ms."""
    from paper_2007_16122_b200 import Batch, Server
    n = 4000
    K = args.topk
    lb = coldgen.make_batch(sch, range(4 * 10**7, 4 * 10**7 + n_requests), n, seed=args.seed + 7)
    hb = Batch(lb.ad_offsets, lb.ids, lb.offs)
    srv = Server(ctx, max_batch_requests=B, max_batch_ads=B * n, top_k=K)
    srv.submit(hb)                        # warm-up (sizes the pinned staging and the library's buffers)
    srv.drain()
    t0 = time.monotonic_ns()
    _, _, done = srv.submit(hb)           # closed loop: everything queued at once
    calls, reqs = srv.drain()
    capacity_rps = n_requests / ((done.max() - t0) / 1e9)
    rows = serve_rates(srv, hb, n, [capacity_rps * f for f in fractions])
    srv.close()
    out = {"requests_per_call_max": B, "requests": n_requests, "ads_per_request": n, "top_k": K,
           "closed_loop": {"ads_per_s": capacity_rps * n, "requests_per_s": capacity_rps, "calls": calls,
                           "requests_per_call": reqs / max(calls, 1)},
           "open_loop": rows,
           "timing": "host CLOCK_MONOTONIC: arrival = the submit time the C replay loop waited for; completion = "
                     "when the dispatcher published the request's top-K to host memory (ids from host memory, one "
                     "H2D and one D2H per coalesced call)"}
    for lim in (1.0, 10.0):
        ok = [r["offered_rps"] for r in rows if r["p99_ms"] <= lim and not r["failed"]]
        out[f"usable_ads_per_s_p99_le_{int(lim)}ms"] = (max(ok) if ok else 0.0) * n
    return out


def run_serve(args):
    """Serving path (P:298 / P:690-692: the paper's GPU was idle between small queries until MPS let them
    share it; "usable QPS"): configs[1]-shaped requests (1 user x 4000 ads, S-paper, fp16, top-500)
    arrive as an open-loop Poisson stream from the host; the cold_server dispatcher coalesces the requests
    that arrived while the GPU was busy into one cold_score_batch + cold_topk call. Latency is end to end
    (host ids in, top-K back in host memory). Reports the closed-loop capacity, p50/p99 per offered rate,
    and the usable rate at p99 <= 1 ms / 10 ms."""
    import torch
    from paper_2007_16122_b200 import Context
    torch.cuda.set_device(0)
    sch = schema_for(args)
    params = coldgen.make_params(sch, seed=args.seed, precision=args.precision)
    B = args.serve_batch
    ctx = Context(sch.groups, sch.k, sch.widths, precision=args.precision, max_ads=B * 4000, max_requests=B)
    load_ctx_params(ctx, params)
    sv = serve_sweep(ctx, sch, args, args.serve_requests, B)
    ctx.close()
    line = {"metric": METRIC, "value": sv["closed_loop"]["ads_per_s"], "unit": "ads/s", "n_gpus": 1,
            "dtype": args.precision, "data": "synthetic (seeded ids, tables, weights)",
            "config": {"workload": f"serving: {args.serve_requests} requests x 4000 ads (BASELINE configs[1] shape), "
                                   f"S-paper, top-{args.topk}; request-coalescing server, <= {B} requests per call; "
                                   f"open-loop Poisson arrivals from the host, end-to-end latency"},
            **sv}
    print(json.dumps(line), flush=True)


def run_latency_sweep(args):
    """SURVEY §8(d) C2 measurements on one B200 (S-paper schema, LL on, K = 500):
    (1) per-request latency vs N (one stream, requests back to back, device events);
    (2) S concurrent streams, each with a cold_ctx_clone over the same parameters, closed loop:
        aggregate ads/s and per-request p99 (the B200 stand-in for the paper's MPS);
    (3) ads/s per compute precision at 512 requests x 4000 ads (Table tab:qps_cuda)."""
    import torch
    from paper_2007_16122_b200 import Batch, Context
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    sch = schema_for(args)
    K = args.topk
    nl = args.latency_requests
    out = {"metric": METRIC, "unit": "ads/s", "n_gpus": 1, "data": "synthetic (seeded ids, tables, weights)",
           "config": {"workload": "BASELINE configs[1] family: 1 user x N ads per request, S-paper, top-500"}}
    params = coldgen.make_params(sch, seed=args.seed, precision="f16")
    ctx = Context(sch.groups, sch.k, sch.widths, precision="f16", max_ads=10000, max_requests=1)
    load_ctx_params(ctx, params)

    def requests(n, count, base):
        lb = coldgen.make_batch(sch, range(base, base + count), n, seed=args.seed + 5)
        return [Batch.from_numpy(b.ad_offsets, b.ids, b.offs) for b in
                (coldgen.sub_batch(lb, [i]) for i in range(count))]

    # (1) latency vs N: >= 10^4 sequential CUDA-graph replays per N (uniform ids), Zipf(1.05) at 4000
    sweep = []
    for n in (300, 1000, 4000, 10000):
        r = graph_latency(ctx, sch, n, nl, K, seed=args.seed + 5 + n, dist="uniform", dev=dev)
        r.pop("timing")
        sweep.append(r)
    r = graph_latency(ctx, sch, 4000, nl, K, seed=args.seed + 5, dist="zipf", dev=dev)
    out["latency_timing"] = r.pop("timing")
    sweep.append(r)
    out["latency_vs_n"] = sweep
    # (2) S streams, closed loop, N = 4000
    n = 4000
    reqs = requests(n, min(nl, 2000), 5 * 10**7)
    ao = np.asarray([0, n], np.int32)
    multi = []
    for S in (1, 4, 8):
        ctxs = [ctx] + [ctx.clone() for _ in range(S - 1)]
        streams = [torch.cuda.Stream() for _ in range(S)]
        bufs = [(torch.empty(n, dtype=torch.float32, device=dev), torch.empty(K, dtype=torch.int32, device=dev),
                 torch.empty(K, dtype=torch.float32, device=dev)) for _ in range(S)]
        per = [reqs[s::S] for s in range(S)]
        for s in range(S):   # warm-up
            with torch.cuda.stream(streams[s]):
                for r in per[s][:3]:
                    ctxs[s].score_request(r, bufs[s][0], stream=streams[s])
                    ctxs[s].topk(bufs[s][0], r.ad_offsets, ao, K, bufs[s][1], bufs[s][2], stream=streams[s])
        torch.cuda.synchronize()
        evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in per[s]]
               for s in range(S)]
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for s in range(S):
            streams[s].wait_event(t0)
        for i in range(max(len(p) for p in per)):   # issue round-robin so the streams run concurrently
            for s in range(S):
                if i < len(per[s]):
                    r = per[s][i]
                    with torch.cuda.stream(streams[s]):
                        evs[s][i][0].record(streams[s])
                        ctxs[s].score_request(r, bufs[s][0], stream=streams[s])
                        ctxs[s].topk(bufs[s][0], r.ad_offsets, ao, K, bufs[s][1], bufs[s][2], stream=streams[s])
                        evs[s][i][1].record(streams[s])
        torch.cuda.synchronize()
        lat = np.array([a.elapsed_time(b) for s in range(S) for a, b in evs[s]])
        total_ms = max(t0.elapsed_time(evs[s][-1][1]) for s in range(S))
        multi.append({"streams": S, "requests": len(reqs), "ads_per_s": len(reqs) * n / (total_ms / 1e3),
                      "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
                      "usable_rps_p99_le_1ms": usable_rate(lat, 1.0, servers=S),
                      "usable_rps_p99_le_10ms": usable_rate(lat, 10.0, servers=S),
                      "usable_note": "S-server open-loop Poisson simulation over the per-request device times "
                                     "measured with S streams busy (conservative at low load)"})
        for c in ctxs[1:]:
            c.close()
    out["multi_stream_n4000"] = multi
    ctx.close()
    # (3) precision table at 512 x 4000
    R, n = 512, 4000
    batch = coldgen.make_batch(sch, range(R), n, seed=args.seed + 1)
    prec_rows = []
    for prec in ("f32", "f16", "bf16"):
        pp = coldgen.make_params(sch, seed=args.seed, precision=prec)
        c = Context(sch.groups, sch.k, sch.widths, precision=prec, max_ads=batch.n_ads, max_requests=R)
        load_ctx_params(c, pp)
        db = Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs)
        sc = torch.empty(batch.n_ads, dtype=torch.float32, device=dev)
        idx = torch.empty(R * K, dtype=torch.int32, device=dev)
        key = torch.empty(R * K, dtype=torch.float32, device=dev)
        for _ in range(2):
            c.score_batch(db, sc)
            c.topk(sc, db.ad_offsets, batch.ad_offsets, K, idx, key)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steps = 3
        for _ in range(steps):
            c.score_batch(db, sc)
            c.topk(sc, db.ad_offsets, batch.ad_offsets, K, idx, key)
        e1.record()
        e1.synchronize()
        prec_rows.append({"precision": prec, "ads_per_s": steps * batch.n_ads / (e0.elapsed_time(e1) / 1e3),
                          "fc_path": "fp32 FFMA (SIMT, no TF32)" if prec == "f32" else "tcgen05 fp32-accumulate"})
        c.close()
        del pp
    out["precision"] = prec_rows
    out["value"] = sweep[2]["ads_per_s"]
    print(json.dumps(out), flush=True)


class RankStep:
    """One bench step on this rank: cold_score_batch over the rank's requests,
    cold_topk into device buffers, and at N > 1 the per-request top-K all-gather (dist.gather_topk:
    NCCL in bench, gloo in the one-GPU multi-process test). The result of a step is
    `result()`: this rank's [r_pad * K] idx / key at N = 1, the rank-major [world * r_pad * K]
    gathered blocks at N > 1 (unpad with dist.unpad_gathered)."""

    def __init__(self, ctx, batch, K, world, r_pad, dev):
        import torch
        from paper_2007_16122_b200 import Batch
        self.ctx, self.batch, self.K, self.world, self.r_pad = ctx, batch, K, world, r_pad
        self.db = Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs, device=dev)
        self.scores = torch.empty(batch.n_ads, dtype=torch.float32, device=dev)
        self.idx = torch.zeros(r_pad * K, dtype=torch.int32, device=dev)
        self.key = torch.zeros(r_pad * K, dtype=torch.float32, device=dev)
        self.g_idx = self.g_key = None
        if world > 1:
            self.g_idx = torch.empty(world * r_pad * K, dtype=torch.int32, device=dev)
            self.g_key = torch.empty(world * r_pad * K, dtype=torch.float32, device=dev)
        self.gather_events = None     # a list: (start, end) CUDA events around every top-K gather

    def result(self):
        return (self.g_idx, self.g_key) if self.world > 1 else (self.idx, self.key)

    def __call__(self, b=None):
        import torch
        from paper_2007_16122_b200.dist import gather_topk
        self.ctx.score_batch(b if b is not None else self.db, self.scores)
        self.ctx.topk(self.scores, self.db.ad_offsets, self.batch.ad_offsets, self.K, self.idx, self.key)
        if self.world > 1:
            ev = None
            if self.gather_events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            gather_topk(self.idx, self.key, self.g_idx, self.g_key)
            if ev is not None:
                ev[1].record()
                self.gather_events.append(ev)


class SplitRequest:
    """F1 (P:248-250 / P:496-498 split one query's ads into parallel inference calls
    and merge the results): this rank scores its slice [floor(g n/G), floor((g+1) n/G)) of one
    request (cold_score_request), keeps its top-K (cold_topk), the G candidate lists are
    all-gathered rank-major, and cold_merge_topk picks the request's top-K over request positions."""

    def __init__(self, ctx, n_full, n_mine, K, world, dev):
        import torch
        self.ctx, self.K, self.world = ctx, K, world
        self.kl = min(K, n_mine)
        self.sscores = torch.empty(max(1, n_mine), dtype=torch.float32, device=dev)
        self.lidx = torch.empty(self.kl, dtype=torch.int32, device=dev)
        self.lkey = torch.empty(self.kl, dtype=torch.float32, device=dev)
        self.cidx = torch.empty(world * self.kl, dtype=torch.int32, device=dev)
        self.ckey = torch.empty(world * self.kl, dtype=torch.float32, device=dev)
        self.midx = torch.empty(K, dtype=torch.int32, device=dev)
        self.mkey = torch.empty(K, dtype=torch.float32, device=dev)
        self.ao_full = np.asarray([0, n_full], np.int32)
        self.d_ao_full = torch.from_numpy(self.ao_full).to(dev)
        self.ao_loc = np.asarray([0, n_mine], np.int32)

    def __call__(self, b):
        from paper_2007_16122_b200.dist import gather_topk
        self.ctx.score_request(b, self.sscores)
        self.ctx.topk(self.sscores, b.ad_offsets, self.ao_loc, self.kl, self.lidx, self.lkey)
        gather_topk(self.lidx, self.lkey, self.cidx, self.ckey)
        self.ctx.merge_topk(self.ckey, self.cidx, self.world, self.kl, self.d_ao_full, self.ao_full, self.K,
                            self.midx, self.mkey)
        return self.midx, self.mkey


def rank_requests(args, world, rank):
    """The rank's share of the configs[4] request stream: strong scaling (default) partitions the
    one stream of args.requests requests into near-equal contiguous blocks; weak
    scaling gives every rank its own block of args.requests."""
    from paper_2007_16122_b200.dist import request_block, split_even
    if args.scaling == "weak":
        return request_block(args.requests, rank), args.requests
    return split_even(args.requests, world, rank), -(-args.requests // world)


def kernel_classes(sch, prof_ms, prof_n, prof_fl, names_extra=None):
    """Per kernel class of the profiled region: launches, average device time, share of the summed
    kernel time, and for the FC classes the algorithmic TFLOP/s (the library counts each launch's
    FLOPs from the rows it covered, so mixed chain / layer-by-layer steps attribute correctly)."""
    from paper_2007_16122_b200.cold import (PROF_CHAIN, PROF_FC, PROF_GATHER, PROF_MLP_F32, PROF_SE_DENSE,
                                            PROF_TAIL, PROF_TOPK, PROF_USER)
    names = {PROF_USER: "user", PROF_GATHER: "gather", PROF_TOPK: "topk", PROF_SE_DENSE: "se_dense",
             PROF_CHAIN: "chain (fc1+fc2+fc3)", PROF_TAIL: "tail (fc4+fc5+head)", PROF_MLP_F32: "mlp_f32 (all layers)"}
    for l in range(len(sch.widths) - 1):
        names[PROF_FC + l] = f"gemm fc{l + 1}" + ("+head" if l == len(sch.widths) - 2 else "")
    fc_kinds = {PROF_CHAIN, PROF_TAIL, PROF_MLP_F32} | {PROF_FC + l for l in range(len(sch.widths) - 1)}
    total = float(prof_ms.sum())
    out = {}
    for kind, name in names.items():
        if not prof_n[kind]:
            continue
        d = {"launches": int(prof_n[kind]), "avg_us": float(prof_ms[kind] / prof_n[kind] * 1e3),
             "share": float(prof_ms[kind] / total), "total_ms": float(prof_ms[kind]), "fc": kind in fc_kinds}
        if prof_fl[kind] > 0:
            d["tflops"] = float(prof_fl[kind] / (prof_ms[kind] / 1e3) / 1e12)
            d["flop_per_launch"] = float(prof_fl[kind] / prof_n[kind])
        out[name] = d
    return out


def load_ncu_summary():
    """profiles/ncu_traffic.json: per-kernel ncu --set full figures of the committed capture (DRAM bytes
    per launch and per ad, tensor-pipe %), with the commit it was taken at."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f)


def fc_roofline(classes, peaks, peak_src, clocks, ncu):
    """Roofline of the dominant FC kernel class (the largest share of the step): algorithmic TFLOP/s
    over its CUDA-event time against the measured bf16 peaks (fp16 runs at the bf16 rate on sm_100):
    `frac` = burst (a plain cuBLAS 8192^3 bf16 GEMM, MEASURED_PEAKS.json), `frac_sustained` = the
    seconds-long loop, and `frac_sustained_at_run_clock` = that sustained figure scaled from the clock
    it was measured at to this run's median SM clock (the kernel's honest fraction when the run sat at
    a higher power-capped clock than the peak measurement). `tensor_active_ncu` is ncu's
    sm__pipe_tensor_cycles_active of the committed capture of the same kernel."""
    fc = {k: v for k, v in classes.items() if v.get("fc")}
    if not fc:
        return None
    name, d = max(fc.items(), key=lambda kv: kv[1]["total_ms"])
    burst = float(peaks.get("bf16_tflops"))
    sus = float(peaks.get("bf16_tflops_sustained", burst))
    sus_mhz = (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")
    run_mhz = (clocks or {}).get("sm_mhz")
    a = d.get("tflops", 0.0)
    r = {"bound": "tensor", "kernel": name, "achieved": a, "peak": burst, "unit": "TFLOP/s", "frac": a / burst,
         "frac_burst": a / burst, "frac_sustained": a / sus, "peak_sustained": sus,
         "peak_source": f"bf16_tflops (burst) {peak_src}; fp16 runs at the bf16 rate",
         "algorithmic": f"{d.get('flop_per_launch', 0):.4g} FLOP per launch (rows x 2 sum(in x out) of the covered "
                        f"layers), avg launch {d['avg_us']:.1f} us"}
    if sus_mhz and run_mhz:
        at_clock = sus * float(run_mhz) / float(sus_mhz)
        r["peak_sustained_at_run_clock"] = at_clock
        r["frac_sustained_at_run_clock"] = a / at_clock
        r["clock_note"] = (f"sustained peak measured at a median {sus_mhz:.0f} MHz; this run's median SM clock "
                           f"{run_mhz:.0f} MHz")
    k = ncu.get("kernels", {}).get(name.split(" ")[0], {})
    r["traffic"] = None
    if k.get("dram_bytes_per_ad") and k.get("flop_per_ad") and d.get("flop_per_launch"):
        # the capture's bytes per ad x this run's ads per launch (FLOPs per launch / FLOPs per ad)
        r["traffic"] = k["dram_bytes_per_ad"] * d["flop_per_launch"] / k["flop_per_ad"]
        r["traffic_note"] = f"ncu dram read+write of the committed capture: {k['dram_bytes_per_ad']:.0f} B/ad"
    r["tensor_active_ncu"] = k.get("tensor_active_pct")
    r["ncu_commit"] = ncu.get("commit")
    bad = [k for k, v in fc.items() if v.get("tflops", 0.0) > 1.2 * sus]
    if bad:
        r["suspect"] = (f"{bad}: above 1.2x the measured sustained peak, i.e. the timed launches did not do "
                        f"the counted work; do not use this line")
    return r


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.latency_sweep:
        run_latency_sweep(args)
        return
    if args.serve:
        run_serve(args)
        return
    if args.vps:
        run_vps(args)
        return
    if args.se_sweep:
        run_se_sweep(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2007_16122_b200 import Batch, Context
    from paper_2007_16122_b200.cold import PROF_GATHER

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # COLD_BENCH_ONE_GPU=1 (path check only, never a bench number): every rank on cuda:0 over gloo, so the
    # N > 1 code path (partition, RankStep, gather, e2e D2H, SplitRequest, per-rank timing) runs on a 1-GPU box
    one_gpu = os.environ.get("COLD_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if one_gpu else dev     # bookkeeping collectives (gloo: host tensors)

    sch = schema_for(args)
    t_setup = time.perf_counter()
    params = coldgen.make_params(sch, seed=args.seed, precision=args.precision)
    reqs, r_pad = rank_requests(args, world, rank)
    batch = coldgen.make_batch(sch, reqs, args.ads, seed=args.seed + 1)
    N = batch.n_ads
    ctx = Context(sch.groups, sch.k, sch.widths, precision=args.precision, device=local, max_ads=N,
                  max_requests=max(batch.R, 1), chunk_ads=args.chunk, se_mode="dense" if args.se_dense else "group",
                  kernel_flags=args.kernel_flags, gather_ring=args.gather_ring, gather_span_chunks=args.gather_span,
                  chain_min_ads=args.chain_min)
    load_ctx_params(ctx, params, dense_se_params(sch, args.seed + 17) if args.se_dense else None)
    K = args.topk
    step = RankStep(ctx, batch, K, world, r_pad, dev)
    stream = torch.cuda.current_stream()
    setup_s = time.perf_counter() - t_setup
    n_all = [N]
    if world > 1:
        t = torch.tensor([N], device=cdev, dtype=torch.int64)
        gl = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gl, t)
        n_all = [int(x.item()) for x in gl]

    def max_over_ranks(ms):
        if world == 1:
            return ms, [ms]
        t = torch.tensor([ms], device=cdev, dtype=torch.float64)
        gl = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gl, t)
        per = [float(x.item()) for x in gl]
        return max(per), per

    def timed(fn, steps, sampler=None, profile=False):
        """W warm-up steps, barrier + sync, `steps` timed steps between CUDA events on the launching
        stream, sync + barrier; returns the max over ranks."""
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if profile:
            ctx.profile(True)
        if sampler:
            sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        prof = None
        if profile:
            prof = ctx.profile_read(with_flop=True)
            ctx.profile(False)
        if world > 1:
            dist.barrier()
        ms, per = max_over_ranks(e0.elapsed_time(e1))
        return ms, per, clocks, prof

    gpu_id = local
    try:
        gpu_id = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    except Exception:
        pass
    sampler = ClockSampler(gpu_id)
    ms, per_rank_ms, clocks, _ = timed(step, args.steps, sampler=sampler)
    ms_step = ms / args.steps
    total_ads = sum(n_all) * args.steps
    value = total_ads / (ms / 1e3)
    # per-kernel device time: the same steps again with a CUDA-event pair around every launch
    # (the library records them on the launching stream); kept out of the `value` region because
    # an event record between kernels serialises their tails.
    step.gather_events = [] if world > 1 else None
    ms_prof, _, _, prof = timed(step, args.steps, profile=True)
    gather_ms = None
    if step.gather_events:
        torch.cuda.synchronize()
        g = sum(a.elapsed_time(b) for a, b in step.gather_events[-args.steps:]) / args.steps
        gather_ms, _ = max_over_ranks(g)
    step.gather_events = None

    peaks, peak_src = measured_peaks()
    prof_ms, prof_n, prof_fl = prof
    info = ctx.info()
    classes = kernel_classes(sch, prof_ms, prof_n, prof_fl)
    ncu = load_ncu_summary()
    roofline = fc_roofline(classes, peaks, peak_src, clocks, ncu)
    gb_per_ad, rows_per_ad = gather_bytes_per_ad(sch, 2 if args.precision != "f32" else 4)
    roofline_gather = None
    if prof_n[PROF_GATHER]:
        hb = float(peaks["hbm_gbs"])
        ga = N * args.steps * gb_per_ad / (prof_ms[PROF_GATHER] / 1e3) / 1e9
        classes["gather"]["gbs"] = ga
        gk = ncu.get("kernels", {}).get("gather", {})
        traffic_g = gk["dram_bytes_per_ad"] * N * args.steps / float(prof_n[PROF_GATHER]) \
            if gk.get("dram_bytes_per_ad") else None
        roofline_gather = {"bound": "hbm", "kernel": "gather", "achieved": ga, "peak": hb, "unit": "GB/s",
                           "frac": ga / hb, "traffic": traffic_g,
                           "traffic_note": "ncu dram read+write bytes per ad of the committed capture "
                                           "(profiles/ncu_traffic.json) x ads per launch: below the algorithmic "
                                           "bytes because L2 serves repeated rows of the column-wise gather",
                           "algorithmic": f"{gb_per_ad:.0f} B/ad ({rows_per_ad:.0f} rows x {sch.k} x 2 B + ids "
                                          f"+ X_ac write)"}
        span_ads = min(N, info["chunk_ads"] * int(info.get("gather_span_chunks", 16) or 16))
        model = gather_access_model(sch, span_ads, 2 if args.precision != "f32" else 4, hb)
        g_ads = N * args.steps / (prof_ms[PROF_GATHER] / 1e3)
        model.update({"achieved_ads_per_s": g_ads,
                      "frac_overlapped": g_ads / model["ceiling_ads_per_s_overlapped"],
                      "frac_serial": g_ads / model["ceiling_ads_per_s_serial"],
                      "note": "random 32 B rows cost 125 DRAM B each and cap at 46 G rows/s on this B200 "
                              "(tools/probes/gather_ceiling.cu, profiles/r01/gather_ceiling.jsonl); ceilings "
                              "from the per-group L2 / DRAM split of the column-wise span, DRAM and L2 time "
                              "overlapped (max) or serial (sum)"})
        roofline_gather["random_access_model"] = model
    fc_ms = sum(v["total_ms"] for v in classes.values() if v.get("fc"))
    fc_flop = sum(v.get("flop_per_launch", 0.0) * v["launches"] for v in classes.values() if v.get("fc"))
    fc_stack = {"tflops": fc_flop / (fc_ms / 1e3) / 1e12 if fc_ms else None,
                "note": "every FC kernel class of the profiled region: algorithmic FLOPs / summed device time"}
    if fc_ms:
        fc_stack["frac_burst"] = fc_stack["tflops"] / float(peaks["bf16_tflops"])
    gpu_launches = int(prof_n.sum())

    # ---- e2e: host (pinned) inputs through the C ABI; the step's top-K (gathered at N > 1) lands in
    # device memory and is read back to pinned host memory inside the timed region ----
    e2e = None
    if not args.no_e2e:
        hb = Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs, pin=True)
        res_idx, res_key = step.result()
        h_idx = torch.empty(res_idx.numel(), dtype=torch.int32).pin_memory()
        h_key = torch.empty(res_key.numel(), dtype=torch.float32).pin_memory()
        reader = rank == 0          # at N > 1 the merged result is consumed on rank 0

        def e2e_step():
            step(hb)
            if reader:
                h_idx.copy_(res_idx, non_blocking=True)
                h_key.copy_(res_key, non_blocking=True)

        ms_e, _, _, _ = timed(e2e_step, args.steps)
        h2d = sum(int(x.nbytes) for x in batch.ids if x is not None) + \
            sum(int(x.nbytes) for x in batch.offs if x is not None) + int(batch.ad_offsets.nbytes)
        d2h = int(h_idx.numel() * 4 + h_key.numel() * 4)
        e2e = {"value": total_ads / (ms_e / 1e3), "unit": "ads/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ms_e / args.steps,
               "note": "per rank: the rank's pinned-host ids staged by the library (H2D inside the timed region); "
                       "top-K to device, gathered over NCCL at N > 1, D2H of the (gathered) top-K on rank 0"}

    # ---- p50 / p99 request latency at configs[1] (1 user x 4000 ads), device-timed ----
    latency = None
    if not args.no_latency and rank == 0:
        nl = args.latency_requests
        # >= 10^4 sequential requests, CUDA-graph replay, uniform and Zipf(1.05) ids
        try:
            latency = graph_latency(ctx, sch, 4000, nl, K, seed=args.seed + 1, dist="uniform", dev=dev)
            latency["zipf"] = {k: v for k, v in graph_latency(ctx, sch, 4000, nl, K, seed=args.seed + 1,
                                                              dist="zipf", dev=dev).items() if k != "timing"}
        except Exception as exc:   # optional section: report, keep the headline line
            latency = {"error": f"{type(exc).__name__}: {exc}"}
        # direct library calls (no graph), requests back to back
        nd = min(nl, 1000)
        lb = coldgen.make_batch(sch, range(10**7, 10**7 + nd), 4000, seed=args.seed + 1)
        singles = [Batch.from_numpy(s.ad_offsets, s.ids, s.offs) for s in
                   (coldgen.sub_batch(lb, [i]) for i in range(nd))]
        lscores = torch.empty(4000, dtype=torch.float32, device=dev)
        lidx = torch.empty(K, dtype=torch.int32, device=dev)
        lkey = torch.empty(K, dtype=torch.float32, device=dev)
        ao = np.asarray([0, 4000], np.int32)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nd)]
        for i in range(min(10, nd)):
            ctx.score_request(singles[i], lscores)
            ctx.topk(lscores, singles[i].ad_offsets, ao, K, lidx, lkey)
        torch.cuda.synchronize()
        for i in range(nd):
            evs[i][0].record(stream)
            ctx.score_request(singles[i], lscores)
            ctx.topk(lscores, singles[i].ad_offsets, ao, K, lidx, lkey)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        lat = np.array([a.elapsed_time(b) for a, b in evs])
        latency["direct_calls"] = {"requests": nd, "p50_ms": float(np.percentile(lat, 50)),
                                   "p99_ms": float(np.percentile(lat, 99)), "mean_ms": float(lat.mean()),
                                   "timing": "device events per request (score + top-500), direct library calls "
                                             "back to back on one stream"}

    # ---- F1: one request's ads split across all ranks (world > 1), per-rank top-K, NCCL all-gather
    # of the candidate lists, cold_merge_topk; p50 / p99 per request at N = args.ads ----
    latency_split = None
    if not args.no_latency and world > 1:
        try:
            from paper_2007_16122_b200.dist import slice_requests
            nl = min(args.latency_requests, 500)
            lb = coldgen.make_batch(sch, range(3 * 10**7, 3 * 10**7 + nl), args.ads, seed=args.seed + 3)
            sides = [g.side for g in sch.groups]
            mine = []
            for i in range(nl):
                one = coldgen.sub_batch(lb, [i])
                ao_s, ids_s, offs_s, _ = slice_requests(one.ad_offsets, one.ids, one.offs, sides, world, rank)
                mine.append(Batch.from_numpy(ao_s, ids_s, offs_s))
            split = SplitRequest(ctx, args.ads, int(ao_s[-1]), K, world, dev)
            for i in range(min(10, nl)):
                split(mine[i])
            torch.cuda.synchronize()
            dist.barrier()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nl)]
            for i in range(nl):
                evs[i][0].record(stream)
                split(mine[i])
                evs[i][1].record(stream)
            torch.cuda.synchronize()
            lat = torch.tensor([a.elapsed_time(b) for a, b in evs], dtype=torch.float64, device=cdev)
            dist.all_reduce(lat, op=dist.ReduceOp.MAX)
            lat = lat.cpu().numpy()
            latency_split = {"n_ads": args.ads, "requests": nl, "gpus": world, "p50_ms": float(np.percentile(lat, 50)),
                             "p99_ms": float(np.percentile(lat, 99)), "mean_ms": float(lat.mean()),
                             "ads_per_s": args.ads / (float(lat.mean()) / 1e3),
                             "timing": "per request, max over ranks of device events: score own slice + top-K, "
                                       "NCCL all-gather of the G candidate lists, cold_merge_topk (F1)"}
        except Exception as exc:   # optional section: report, keep the headline line
            latency_split = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- serving: the coalescing server (D-13) on this context, configs[1]-shaped requests, open loop ----
    serve = None
    if rank == 0 and world == 1 and not args.no_latency and not args.no_serve:
        try:
            serve = serve_sweep(ctx, sch, args, 2000, args.serve_batch, fractions=(0.25, 0.5, 0.75, 0.9))
        except Exception as exc:   # optional section: report, keep the headline line
            serve = {"error": f"{type(exc).__name__}: {exc}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(sch, params, batch)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "ads/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic (seeded ids, tables, weights)",
            "config": config_dict(args, sch, world),
            "roofline": roofline, "roofline_gather": roofline_gather, "fc_stack": fc_stack,
            "kernels": classes, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
            "clocks": clocks, "latency": latency, "latency_split": latency_split, "serve": serve, "setup_s": setup_s,
            "compressed_activations": bool(info.get("compressed_activations", 0)),
            "profiled_region": {"ms_per_step": ms_prof / args.steps,
                                "note": "per-kernel CUDA events (kernels, roofline) come from this second timed "
                                        "region of the same steps"},
        }
        if world > 1:
            line["ranks"] = {"ads_per_rank": n_all, "ms_per_step_per_rank": [m / args.steps for m in per_rank_ms],
                             "imbalance_max_over_min": max(per_rank_ms) / min(per_rank_ms),
                             "topk_gather_ms_per_step": gather_ms,
                             "gather_note": "max over ranks of CUDA events around the NCCL all-gather of the "
                                            "per-request top-K (profiled region)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
