python -m paper_2007_16122_b200.build >/dev/null
timeout 900 python bench.py --se-sweep > gpurun_out/se_sweep_r01j.jsonl 2> gpurun_out/se_sweep_r01j.err
