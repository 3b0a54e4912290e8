"""chain_kernel wait cycles per role (-DCOLD_INSTRUMENT build, tools/ab_build.sh): kcycles per CTA over one scoring call."""
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
ms = e0.elapsed_time(e1)
v = buf[32:46].astype(np.float64)
names = ["prod_empty", "prod_hready", "mma_full", "mma_tempty", "mma_uxfull", "epi_tfull(sum of 8 warps)",
         "mma_issuer_elapsed", "-", "mma_full_fc1", "mma_full_fc2", "mma_full_fc3", "mma_tempty_fc1", "mma_tempty_fc2",
         "mma_tempty_fc3"]
ctas = 148.0
print(f"call {ms:.2f} ms = {ms * 1.92e3:.0f} kcycles at 1.92 GHz; per CTA (leader-only for MMA rows: /74):")
for i, n in enumerate(names):
    if n == "-":
        continue
    div = 74.0 if i in (2, 3, 4) or i >= 6 else ctas
    print(f"  {n}: {v[i] / div / 1e3:.1f} kcycles")

# epilogue sections per layer (sum over the 8 epilogue warps' lane 0, per CTA): TMEM load + wait, math + pack,
# wait for the staging box, smem writes, store issue, proxy fence, group barrier after the writes
sec = ["tmem_ld", "math", "box_wait", "sts", "store", "fence", "group_bar"]
for l in range(3):
    v = buf[48 + 8 * l:48 + 8 * l + 7].astype(np.float64) / ctas / 8 / 1e3
    print(f"  epilogue fc{l + 1} per warp (kcycles): " + ", ".join(f"{n} {x:.1f}" for n, x in zip(sec, v)))
