#!/bin/bash
# Run under gpurun: launch list + one `--set full` capture of each hot kernel, then
# profiles-ready summaries (gpurun_out/ncu_summary_<tag>.txt, gpurun_out/ncu_traffic_<tag>.json).
# Usage: bash tools/ncu_profile.sh <tag> [kernels...]   (default: gather chain tail45)
set -x
TAG=${1:-r02}
shift
KERNELS=${@:-gather chain tail45}
OUT=gpurun_out
# 256 requests x 9472 ads = 16 full 151552-ad chunks per step (one 16-chunk gather span)
ARGS=${NCU_ARGS:-"--requests 256 --ads 9472 --steps 2 --warmup 1 --no-e2e --no-latency --no-cpu"}
python -m paper_2007_16122_b200.build >/dev/null
# 1. launch list (cold-cache, serialised: compare shares)
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py $ARGS > $OUT/ncu_launch_bench_$TAG.log 2>&1
REPS=""
for k in $KERNELS; do
  case $k in
    gather) RX="regex:gather_kernel"; S=2; C=2; NM=gather;;   # the span's two launches (cross-bag columns, the rest)
    chain) RX="regex:chain_kernel"; S=1; NM=chain;;
    fc1) RX="regex:gemm_pair_kernel"; S=3; NM=fc1;;      # pair launches per chunk: FC1, FC2, FC3
    fc2) RX="regex:gemm_pair_kernel"; S=4; NM=fc2;;
    fc3) RX="regex:gemm_pair_kernel"; S=5; NM=fc3;;
    tail45) RX="regex:tail45_kernel"; S=1; NM=tail;;
    *) RX="regex:$k"; S=1; NM=$k;;
  esac
  C=${C:-1}
  timeout 400 ncu --set full --clock-control none --import-source on -k $RX -s $S -c $C \
    -o $OUT/prof_${k}_$TAG python bench.py $ARGS > $OUT/ncu_${k}_$TAG.log 2>&1
  REPS="$REPS $NM=$OUT/prof_${k}_$TAG.ncu-rep"
  unset C
done
for f in $OUT/prof_*_$TAG.ncu-rep; do python tools/ncu_summary.py $f; done > $OUT/ncu_summary_$TAG.txt 2>&1
python tools/ncu_traffic.py --commit "${GIT_SHA:-unknown}" --source "ncu --set full, bench.py $ARGS, tag $TAG" \
  --ads chain=151552 --ads tail=151552 --ads gather=2424832 \
  --flop-per-ad chain=1835008 --flop-per-ad tail=82176 --out $OUT/ncu_traffic_$TAG.json $REPS > /dev/null 2>&1
ls -la $OUT
