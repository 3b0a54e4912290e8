set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "server or ring or gathers_bit_exact or paper_stack or variants" > gpurun_out/gpu_tests_r02h.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02h.log
run() { tag=$1; shift; timeout 300 python bench.py --no-latency --no-e2e --no-cpu --steps 5 "$@" > gpurun_out/ab_h_$tag.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab_h_$tag.jsonl').read().splitlines()[-1]);k=d['kernels']
print('$tag', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"; }
for i in 1 2; do
  unset COLD_LIB_AB; run split$i; run onelaunch$i --gather-ring -1
  COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/oldgk.so run oldgk$i --gather-ring -1
done
unset COLD_LIB_AB
for b in 8 32; do timeout 600 python bench.py --serve --serve-batch $b > gpurun_out/serve_r02h_b$b.jsonl 2>&1; tail -c 600 gpurun_out/serve_r02h_b$b.jsonl; done
