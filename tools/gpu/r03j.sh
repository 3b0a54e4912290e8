set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03j.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03j.log
for i in 1 2; do
for f in 0 128; do
  timeout 300 python bench.py --no-latency --no-e2e --no-cpu --no-serve --steps 5 --kernel-flags $f > gpurun_out/ab_tt_${f}_$i.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab_tt_${f}_$i.jsonl').read().splitlines()[-1]);k=d['kernels']
print('$f', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"
done
done
