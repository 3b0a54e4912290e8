set -x
timeout 300 ./tools/probes/gather4_probe > gpurun_out/gather4_probe.jsonl 2>&1; echo probe rc=$?
cat gpurun_out/gather4_probe.jsonl
python -m paper_2007_16122_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_r02e.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests_r02e.log
