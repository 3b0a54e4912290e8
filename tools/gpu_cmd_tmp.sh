python -m paper_2007_16122_b200.build >/dev/null
COLD_USER_FORK=2 timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/gpu_tests_s19.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s19.log
for v in 1 2 1 2; do COLD_USER_FORK=$v timeout 600 python bench.py --latency-sweep --latency-requests 3000 > gpurun_out/lat_s19_$v.jsonl 2>&1; python -c "
import json; L=[json.loads(x) for x in open('gpurun_out/lat_s19_$v.jsonl') if x.startswith('{')][0]
print('fork=$v', [(r['n_ads'], r['ids'], round(r['p50_ms'],4), round(r['p99_ms'],4)) for r in L['latency_vs_n']])" >> gpurun_out/lat_s19.txt 2>&1; done
