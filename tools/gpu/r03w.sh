set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python bench.py --latency-sweep --latency-requests 5000 > gpurun_out/latency_sweep_r03w.jsonl 2> gpurun_out/latency_sweep_r03w.err; echo lat rc=$?
tail -3 gpurun_out/latency_sweep_r03w.err
