"""Print the key numbers of bench JSON lines: python tools/show.py gpurun_out/sweep_*.log"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", open(f).read()[-600:])
        continue
    ks = {k: (round(v["avg_us"], 1), round(v.get("tflops", v.get("gbs", 0)))) for k, v in d.get("kernels", {}).items()}
    print(f.split("/")[-1], f"{d['value'] / 1e6:.1f} Mads/s", f"{d['ms_per_step']:.2f} ms/step",
          "e2e", None if not d.get("e2e") else f"{d['e2e']['value'] / 1e6:.1f}", ks)
