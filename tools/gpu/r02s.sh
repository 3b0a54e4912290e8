set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_r02s.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02s.log
run() { tag=$1; shift; timeout 300 python bench.py --no-latency --no-e2e --no-cpu --steps 5 "$@" > gpurun_out/ab_s_$tag.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab_s_$tag.jsonl').read().splitlines()[-1]);k=d['kernels']
print('$tag', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"; }
for i in 1 2; do run slab$i; run rows$i --kernel-flags 1024; done
