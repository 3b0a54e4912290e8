import numpy as np, torch, sys, json
sys.path.insert(0, '.')
import coldgen
from paper_2007_16122_b200 import Batch, Context
from paper_2007_16122_b200.cold import PROF_FC, PROF_GATHER, PROF_TOPK, PROF_USER
import bench
sch = coldgen.schema_paper()
params = coldgen.make_params(sch, seed=1234, precision="f16")
ctx = Context(sch.groups, sch.k, sch.widths, precision="f16", max_ads=10000, max_requests=1)
bench.load_ctx_params(ctx, params)
for n in (300, 4000, 10000):
    lb = coldgen.make_batch(sch, range(50), n, seed=3)
    reqs = [Batch.from_numpy(b.ad_offsets, b.ids, b.offs) for b in (coldgen.sub_batch(lb, [i]) for i in range(50))]
    sc = torch.empty(n, device="cuda"); K = min(500, n)
    idx = torch.empty(K, dtype=torch.int32, device="cuda"); key = torch.empty(K, device="cuda")
    ao = np.asarray([0, n], np.int32)
    for r in reqs[:5]:
        ctx.score_request(r, sc); ctx.topk(sc, r.ad_offsets, ao, K, idx, key)
    torch.cuda.synchronize()
    ctx.profile(True)
    for r in reqs:
        ctx.score_request(r, sc); ctx.topk(sc, r.ad_offsets, ao, K, idx, key)
    torch.cuda.synchronize()
    ms, cnt = ctx.profile_read()
    ctx.profile(False)
    out = {k: (round(float(ms[k]) / 50 * 1e3, 2), int(cnt[k]) // 50) for k in range(len(ms)) if cnt[k]}
    print(n, json.dumps(out), "total_us", round(float(ms.sum()) / 50 * 1e3, 1))
