set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python bench.py --latency-sweep --latency-requests 5000 > gpurun_out/latency_sweep_r02w.jsonl 2> gpurun_out/latency_sweep_r02w.err; echo lat rc=$?
timeout 900 python bench.py --se-sweep --steps 3 --warmup 2 > gpurun_out/se_sweep_r02w.jsonl 2> gpurun_out/se_sweep_r02w.err; echo se rc=$?
timeout 600 python bench.py --vps --steps 5 > gpurun_out/vps_r02w.jsonl 2> gpurun_out/vps_r02w.err; echo vps rc=$?
timeout 900 python bench.py --se-dense --requests 2048 --steps 3 --no-latency --no-cpu --no-e2e > gpurun_out/bench_se_dense_r02w.jsonl 2> gpurun_out/se_dense_r02w.err; echo sed rc=$?
