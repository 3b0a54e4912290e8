set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "server" > gpurun_out/gpu_tests_r02g.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gpu_tests_r02g.log
timeout 600 python bench.py --serve > gpurun_out/serve_r02g.jsonl 2> gpurun_out/serve_r02g.err; echo serve rc=$?
tail -c 2500 gpurun_out/serve_r02g.jsonl; tail -5 gpurun_out/serve_r02g.err
bash tools/gpu/ab_multi.sh gk paper_2007_16122_b200/_ab/fields.so paper_2007_16122_b200/_ab/oldgk.so paper_2007_16122_b200/_ab/old.so
