set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 300 ncu --set full --import-source on --clock-control none -k regex:topk_small -c 1 -o gpurun_out/prof_topk_r03d python tools/probes/lat_ncu.py 4000 2 > gpurun_out/prof_topk_r03d.log 2>&1; echo ncu rc=$?
