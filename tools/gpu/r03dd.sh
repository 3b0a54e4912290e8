set -x
python -m paper_2007_16122_b200.build > /dev/null
for i in 1 2; do
for sp in 16 1 2 4; do
  timeout 300 python bench.py --no-latency --no-e2e --no-cpu --no-serve --steps 5 --gather-span $sp > gpurun_out/ab_span_${sp}_$i.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab_span_${sp}_$i.jsonl').read().splitlines()[-1]);k=d['kernels']
print('span$sp', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"
done
done
