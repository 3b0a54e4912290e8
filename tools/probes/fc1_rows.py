"""Which rows of the paper-stack parity case are off (u1-MMA debugging)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.fixtures import small_case
from tests.gpu_helpers import make_ctx, gpu_scores, rel_err
import oracle
for prec in ("f16",):
    sch, params, batch = small_case("paper", R=4, n_ads=(1000, 129, 1, 700), precision=prec, cap=50000, seed=31)
    ctx = make_ctx(sch, params)
    p, z = oracle.score(oracle.Model(sch, params), batch)
    got = gpu_scores(ctx, batch)
    err = rel_err(got, p)
    bad = np.where(err > 2e-3)[0]
    print(prec, "bad rows:", len(bad), bad[:40], "...", bad[-20:])
    print("err by 128-row tile:", [float(np.round(err[i:i+128].max(), 4)) for i in range(0, len(err), 128)])
