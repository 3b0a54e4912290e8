set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/lat_launches_warm_r03o.csv python tools/probes/lat_ncu.py 4000 8 > gpurun_out/lat_ncu_r03o.log 2>&1; echo ncu rc=$?
