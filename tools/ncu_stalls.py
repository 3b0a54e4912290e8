"""Per-source-line stall breakdown from `ncu -i rep --page source --csv --print-source cuda`.
usage: python tools/ncu_stalls.py <rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
agg = {}
file = ""
func = ""
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        file = r[1].split("/")[-1]
    if len(r) == 2 and r[0] == "Function Name":
        if func and r[1] != func:
            break            # first kernel only
        func = r[1]
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        if r[3].strip() != "-":      # SASS row (source rows carry the per-line aggregate)
            continue
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        if samp == 0:
            continue
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = int(r[i] or 0)
                except ValueError:
                    v = 0
                if v:
                    stalls[h[6:]] = v
        key = f"{file}:{r[0]}"
        a = agg.setdefault(key, [0, r[1].strip()[:80], {}])
        a[0] += samp
        for k, v in stalls.items():
            a[2][k] = a[2].get(k, 0) + v
tot = sum(v[0] for v in agg.values())
print(func[:120])
print("total samples", tot)
for k, (s, src, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st_s = " ".join(f"{n}={v}" for n, v in sorted(st.items(), key=lambda x: -x[1])[:4])
    print(f"{100 * s / tot:5.1f}% {k:24s} {src:70s} [{st_s}]")
