"""Write profiles/ncu_traffic.json from `ncu --set full` captures of the hot kernels (one launch each):
per kernel, DRAM read+write bytes per launch and per ad, the tensor-pipe and DRAM throughput %, and
the commit the capture was taken at. bench.py reads it for the roofline `traffic` / `tensor_active_ncu`.

  python tools/ncu_traffic.py --commit <sha> --ads chain=151552 --ads gather=303104 --ads tail=151552 \
      --flop-per-ad chain=1835008 --flop-per-ad tail=82176 chain=<rep> gather=<rep> tail=<rep>
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402


UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def num(v):
    parts = str(v).split()
    x = float(parts[0].replace(",", ""))
    return x * UNIT.get(parts[1], 1.0) if len(parts) > 1 else x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--commit", required=True)
    ap.add_argument("--ads", action="append", default=[], help="name=ads per launch")
    ap.add_argument("--flop-per-ad", action="append", default=[], help="name=algorithmic FLOP per ad")
    ap.add_argument("--out", default="profiles/ncu_traffic.json")
    ap.add_argument("--source", default="")
    ap.add_argument("reps", nargs="+", help="name=path.ncu-rep")
    a = ap.parse_args()
    ads = {k: float(v) for k, v in (x.split("=") for x in a.ads)}
    fpa = {k: float(v) for k, v in (x.split("=") for x in a.flop_per_ad)}
    out = {"commit": a.commit, "source": a.source, "kernels": {}}
    for item in a.reps:
        name, rep = item.split("=", 1)
        launches = summary(rep)   # one or more consecutive launches of the kernel class (e.g. the two gather
        #                           launches of one span: the cross-bag columns, then the rest), summed
        rd = sum(num(d["dram__bytes_read.sum"]) for d in launches)
        wr = sum(num(d["dram__bytes_write.sum"]) for d in launches)
        durs = [num(d.get("gpu__time_duration.sum", "0")) for d in launches]
        tot = sum(durs) or 1.0

        def wavg(key):
            return sum(num(d.get(key, "0")) * w for d, w in zip(launches, durs)) / tot
        k = {"kernel_name": " + ".join(d.get("Kernel Name", "").replace("void ", "").split("(")[0] for d in launches),
             "launches": len(launches), "dram_read_bytes": rd, "dram_write_bytes": wr,
             "dram_bytes_per_launch": rd + wr, "duration": " + ".join(d.get("gpu__time_duration.sum") for d in launches),
             "tensor_active_pct": wavg("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
             "dram_throughput_pct": wavg("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
             "l2_throughput_pct": wavg("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
             "warps_active_pct": wavg("sm__warps_active.avg.pct_of_peak_sustained_active")}
        if name in ads:
            k["ads_per_launch"] = ads[name]
            k["dram_bytes_per_ad"] = (rd + wr) / ads[name]
        if name in fpa:
            k["flop_per_ad"] = fpa[name]
        out["kernels"][name] = k
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
