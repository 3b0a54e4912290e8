set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "ring or gathers_bit_exact or paper_stack" > gpurun_out/gpu_tests_r02d.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02d.log
for r in 0 4 5 8 0; do
  COLD_GATHER_RING=$r timeout 300 python bench.py --no-latency --no-e2e --no-cpu --steps 5 > gpurun_out/bench_r02d_ring$r.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/bench_r02d_ring$r.jsonl').read().splitlines()[-1]);k=d['kernels'];print('ring $r', round(d['value']/1e6,1), 'gather_us', round(k['gather']['avg_us'],1), 'chain_us', round(k['chain (fc1+fc2+fc3)']['avg_us'],1), d['clocks']['sm_mhz'])"
done
