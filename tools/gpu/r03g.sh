set -x
python -m paper_2007_16122_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r03g.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_r03g.log
for v in main rb4 rb8; do
  if [ $v = main ]; then unset COLD_LIB_AB; else export COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/$v.so; fi
  timeout 300 python tools/probes/lat_ab.py 0 4000 3000 > gpurun_out/lat_ab_r03g_$v.jsonl 2>&1
done
unset COLD_LIB_AB
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_r03g.csv python tools/probes/lat_ncu.py 4000 3 > gpurun_out/lat_ncu_r03g.log 2>&1; echo ncu rc=$?
