set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_r02l.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02l.log
for i in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --steps 5 --latency-requests 5000 > gpurun_out/bench_r02l_$i.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/bench_r02l_$i.jsonl').read().splitlines()[-1]);k=d['kernels'];l=d['latency']
print('run', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'], 'lat', round(l['p50_ms'],4), round(l['p99_ms'],4))"
done
