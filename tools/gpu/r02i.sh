set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "server or ring" > gpurun_out/gpu_tests_r02i.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02i.log
for b in 1 4 8 32; do timeout 600 python bench.py --serve --serve-batch $b > gpurun_out/serve_r02i_b$b.jsonl 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/serve_r02i_b$b.jsonl').read().splitlines()[-1])
print('b$b', d['closed_loop']); [print('  ', round(r['offered_ads_per_s']/1e6,1), round(r['p50_ms'],3), round(r['p99_ms'],3)) for r in d['open_loop']]"; done
