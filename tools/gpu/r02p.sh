set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multi_rank_gpu.py -q -x -k "topk or split or server or config0 or worked or bench_rank" > gpurun_out/gpu_tests_r02p.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02p.log
for i in 1 2; do
  for v in main nosort; do
    if [ $v = nosort ]; then export COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/nosort.so; else unset COLD_LIB_AB; fi
    timeout 300 python bench.py --requests 64 --steps 3 --warmup 3 --no-e2e --no-cpu --latency-requests 5000 > gpurun_out/lat_r02p_$v$i.jsonl 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/lat_r02p_$v$i.jsonl').read().splitlines()[-1]);l=d['latency']
print('$v', round(l['p50_ms'],4), round(l['p99_ms'],4), 'zipf', round(l['zipf']['p99_ms'],4), 'direct', round(l['direct_calls']['p50_ms'],4))"
  done
done
unset COLD_LIB_AB
timeout 300 python tools/probes/latency_profile.py > gpurun_out/latency_profile_r02p.txt 2>&1; cat gpurun_out/latency_profile_r02p.txt
