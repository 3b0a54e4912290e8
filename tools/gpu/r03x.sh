set -x
COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/xr2.so timeout 300 python -m pytest tests -m gpu -x -q -k "chain or paper_stack or variant" > gpurun_out/gpu_tests_r03x_xr2.log 2>&1; echo xr2 tests rc=$?; tail -2 gpurun_out/gpu_tests_r03x_xr2.log
bash tools/gpu/ab_multi.sh xr paper_2007_16122_b200/_ab/xr2.so
