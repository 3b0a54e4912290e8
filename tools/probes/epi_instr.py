"""Epilogue section timing of the CTA-pair GEMMs (-DCOLD_INSTRUMENT build, tools/ab_build.sh): per epilogue warp, kcycles spent in
[TMEM load+wait, math+pack, staging-buffer wait, smem write+fence, store issue] over one scoring call."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import coldgen  # noqa: E402
from paper_2007_16122_b200 import Batch, Context, lib  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sch = coldgen.schema_paper()
params = coldgen.make_params(sch, seed=1, precision="f16")
batch = coldgen.make_batch(sch, R, 10000, seed=2)
ctx = Context(sch.groups, sch.k, sch.widths, precision="f16", max_ads=batch.n_ads, max_requests=R)
ctx.load_params([t.view(np.uint16) for t in params.tables], params.se_w, params.se_b, params.fc_w, params.fc_b,
                table_dtype="f16")
db = Batch.from_numpy(batch.ad_offsets, batch.ids, batch.offs)
out = torch.empty(batch.n_ads, device="cuda")
L = lib()
L.cold_debug_instr.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(8 * 16, np.uint64)
ctx.score_batch(db, out)
torch.cuda.synchronize()
L.cold_debug_instr(buf.ctypes.data, len(buf))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.score_batch(db, out)
e1.record()
torch.cuda.synchronize()
L.cold_debug_instr(buf.ctypes.data, len(buf))
warps = 148 * 8
names = ["tmem_ld", "math", "buf_wait", "sts_fence", "store"]
print(f"call {e0.elapsed_time(e1):.2f} ms for {batch.n_ads} ads")
for l in range(3):
    v = buf[8 * l:8 * l + 5].astype(np.float64) / warps / 1e3
    print(f"layer {l}: " + " ".join(f"{n}={x:.1f}k" for n, x in zip(names, v)) + f" total={v.sum():.1f}k cycles/warp")
