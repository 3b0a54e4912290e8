python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not full_size" > gpurun_out/gpu_tests_s41.log 2>&1
BENCH_ARGS="--requests 1024 --no-e2e --no-latency --no-cpu --steps 5" timeout 1200 bash tools/sweep.sh s41:COLD_TAIL=2 s41old:"COLD_TAIL_REV=0 COLD_SPAN_REV=0 COLD_H3_EF=1" s41ef:COLD_H3_EF=1 s41norev:COLD_SPAN_REV=0
python tools/show.py gpurun_out/sweep_s41*.log > gpurun_out/sweep_s41.txt 2>&1
