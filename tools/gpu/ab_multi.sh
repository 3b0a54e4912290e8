# A/B of the current build against prebuilt variants: bash tools/gpu/ab_multi.sh <tag> <alt1.so> <alt2.so> ...
set -x
TAG=$1; shift
python -m paper_2007_16122_b200.build > /dev/null
for i in 1 2; do
  for v in main "$@"; do
    if [ $v = main ]; then unset COLD_LIB_AB; else export COLD_LIB_AB=$PWD/$v; fi
    n=$(basename $v .so)
    timeout 300 python bench.py --no-latency --no-e2e --no-cpu --steps 5 > gpurun_out/ab_${TAG}_$n$i.jsonl 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_$n$i.jsonl').read().splitlines()[-1]);k=d['kernels']
print('$n', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"
  done
done
unset COLD_LIB_AB
