python -m paper_2007_16122_b200.build >/dev/null
COLD_INSTR=1 python tools/probes/epi_instr.py 128 > gpurun_out/epi_instr.log 2>&1
python -m pytest tests -m gpu -x -q -k "vps or merge or se_stats" > gpurun_out/gpu_tests_s18.log 2>&1
