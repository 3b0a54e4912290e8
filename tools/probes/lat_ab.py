"""Latency A/B of kernel selections on the configs[1] request (1 user x 4000 ads + top-500), graph replay
(bench.graph_latency): python tools/probes/lat_ab.py FLAGS[,FLAGS...] [n_ads] [requests]"""
import json
import sys
import torch
sys.path.insert(0, '.')
import coldgen
from paper_2007_16122_b200 import Context
import bench

flags = [int(f) for f in (sys.argv[1] if len(sys.argv) > 1 else "0").split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
count = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
sch = coldgen.schema_paper()
params = coldgen.make_params(sch, seed=1234, precision="f16")
for rep in range(2):
    for f in flags:
        ctx = Context(sch.groups, sch.k, sch.widths, precision="f16", max_ads=10000, max_requests=4, kernel_flags=f)
        bench.load_ctx_params(ctx, params)
        r = bench.graph_latency(ctx, sch, n, count, 500, 77, dev=torch.device("cuda"))
        print(json.dumps({"flags": f, "rep": rep, "n": n, "p50_us": round(r["p50_ms"] * 1e3, 2),
                          "p99_us": round(r["p99_ms"] * 1e3, 2), "replay_ok": r["replay_matches_direct_call"]}), flush=True)
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
