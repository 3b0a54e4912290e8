set -x
python -m paper_2007_16122_b200.build > /dev/null
for cm in 0 1 0 1; do
  timeout 300 python bench.py --requests 64 --steps 3 --warmup 3 --no-e2e --no-cpu --chain-min $cm --latency-requests 5000 > gpurun_out/lat_r02j_cm$cm.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/lat_r02j_cm$cm.jsonl').read().splitlines()[-1]);l=d['latency']
print('chain_min $cm', round(l['p50_ms'],4), round(l['p99_ms'],4), 'zipf', round(l['zipf']['p99_ms'],4), 'direct', round(l['direct_calls']['p50_ms'],4))"
done
