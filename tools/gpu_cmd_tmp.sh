python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01k.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r01k.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_r01k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01k.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r01k.log
