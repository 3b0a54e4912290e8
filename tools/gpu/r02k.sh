set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "topk or split or config0 or server" > gpurun_out/gpu_tests_r02k.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02k.log
for i in 1 2; do
  timeout 300 python bench.py --requests 64 --steps 3 --warmup 3 --no-e2e --no-cpu --latency-requests 5000 > gpurun_out/lat_r02k_$i.jsonl 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/lat_r02k_$i.jsonl').read().splitlines()[-1]);l=d['latency']
print('lat', round(l['p50_ms'],4), round(l['p99_ms'],4), 'zipf', round(l['zipf']['p99_ms'],4), 'direct', round(l['direct_calls']['p50_ms'],4))"
done
timeout 300 python tools/probes/latency_profile.py > gpurun_out/latency_profile_r02k.txt 2>&1; cat gpurun_out/latency_profile_r02k.txt
