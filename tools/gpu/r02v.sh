set -x
python -m paper_2007_16122_b200.build > /dev/null
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_r02v.jsonl 2> gpurun_out/bench_r02v.err; echo bench rc=$? seconds=$(( $(date +%s) - t0 ))
python -c "
import json;d=json.loads(open('gpurun_out/bench_r02v.jsonl').read().splitlines()[-1]);print(round(d['value']/1e6,1), d['serve']['closed_loop'], [(round(r['offered_ads_per_s']/1e6), round(r['p99_ms'],3)) for r in d['serve']['open_loop']], d['latency']['p99_ms'])"
bash tools/gpu/ab_multi.sh apt paper_2007_16122_b200/_ab/apt8.so
