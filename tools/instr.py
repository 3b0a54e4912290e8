"""Run a short scoring loop in the -DCOLD_INSTRUMENT build and print the GEMM pipeline wait cycles per layer.
usage (GPU): bash tools/ab_build.sh instr -DCOLD_INSTRUMENT; COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/instr.so python tools/instr.py [requests]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import coldgen  # noqa: E402
from paper_2007_16122_b200 import Batch, Context, lib  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 256
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
for _ in range(2):
    ctx.score_batch(db, out)
torch.cuda.synchronize()
L.cold_debug_instr(buf.ctypes.data, len(buf))
ctx.score_batch(db, out)
torch.cuda.synchronize()
L.cold_debug_instr(buf.ctypes.data, len(buf))
names = ["prod_empty", "mma_full", "mma_tempty", "mma_bres", "epi_tfull", "epi_u1", "epi_warps", "prod_total"]
for l in range(2):
    v = buf[8 * l:8 * l + 8].astype(np.float64)
    ctas = v[6] / 8 if v[6] else 1
    print(f"layer {l}: " + " ".join(f"{n}={v[i] / ctas / 1e3:.1f}k" for i, n in enumerate(names) if i != 6),
          f"(per CTA, kcycles; epi per warp x8)")
