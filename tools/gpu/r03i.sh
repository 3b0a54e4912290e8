set -x
python -m paper_2007_16122_b200.build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ts tools/probes/umma_ts_probe.cu && timeout 60 /tmp/ts > gpurun_out/umma_ts_r03i.txt 2>&1; echo ts rc=$?
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tsp tools/probes/umma_ts_pair_probe.cu && timeout 60 /tmp/tsp >> gpurun_out/umma_ts_r03i.txt 2>&1; echo tsp rc=$?
timeout 900 python bench.py > gpurun_out/bench_r03i.jsonl 2> gpurun_out/bench_r03i.err; echo bench rc=$?
