set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -rw > gpurun_out/gpu_tests_r03aa.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests_r03aa.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r03aa.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_r03aa.log
