# end-of-round evidence at HEAD (round 3 tags): tests, smoke, bench, reference arm, serve, ncu captures,
# latency launch lists (cold and warm L2)
export TAG=${TAG:-r03z}
export GIT_SHA=${GIT_SHA:-83fd9d1}
bash tools/gpu/r02_final.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_${TAG}.csv python tools/probes/lat_ncu.py 4000 3 > /dev/null 2>&1; echo latncu rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/lat_launches_warm_${TAG}.csv python tools/probes/lat_ncu.py 4000 8 > /dev/null 2>&1; echo latncuw rc=$?
