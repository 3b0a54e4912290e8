# end-of-round evidence at HEAD: GPU tests, smoke, bench (ours + reference arm), serve sweep, ncu captures
set -x
TAG=${TAG:-r02z}
python -m paper_2007_16122_b200.build > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_${TAG}.txt
timeout 1500 python -m pytest tests -m gpu -q -rw > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests rc=$?
tail -4 gpurun_out/gpu_tests_${TAG}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
cat gpurun_out/smoke_${TAG}.log | tail -3
timeout 900 python bench.py > gpurun_out/bench_${TAG}.jsonl 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.jsonl 2> gpurun_out/bench_ref_${TAG}.err; echo ref rc=$?
timeout 600 python bench.py --serve --serve-batch 32 > gpurun_out/serve_${TAG}.jsonl 2>&1; echo serve rc=$?
GIT_SHA=$GIT_SHA bash tools/ncu_profile.sh ${TAG} > gpurun_out/ncu_profile_${TAG}.log 2>&1; echo ncu rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_${TAG}.jsonl').read().splitlines()[-1]);k=d['kernels']
print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks'], d['roofline']['frac'], d['latency']['p99_ms'])"
