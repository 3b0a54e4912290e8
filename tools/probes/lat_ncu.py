"""One configs[1] request (1 user x N ads + top-500) through direct library calls, a few times: run under
`ncu --metrics gpu__time_duration.sum` to get the per-kernel device times of the latency path without
event overhead, and without ncu for the replayed-graph total."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import coldgen
from paper_2007_16122_b200 import Batch, Context
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sch = coldgen.schema_paper()
params = coldgen.make_params(sch, seed=1234, precision="f16")
ctx = Context(sch.groups, sch.k, sch.widths, precision="f16", max_ads=10000, max_requests=1)
bench.load_ctx_params(ctx, params)
lb = coldgen.make_batch(sch, range(reps), n, seed=3)
reqs = [Batch.from_numpy(b.ad_offsets, b.ids, b.offs) for b in (coldgen.sub_batch(lb, [i]) for i in range(reps))]
sc = torch.empty(n, device="cuda"); K = min(500, n)
idx = torch.empty(K, dtype=torch.int32, device="cuda"); key = torch.empty(K, device="cuda")
ao = np.asarray([0, n], np.int32)
for r in reqs:
    ctx.score_request(r, sc); ctx.topk(sc, r.ad_offsets, ao, K, idx, key)
torch.cuda.synchronize()
print("ok", n, reps)
