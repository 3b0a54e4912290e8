# A/B of the current build against a prebuilt libcold variant: bash tools/gpu/ab_lib.sh <tag> <alt.so> [bench args]
set -x
TAG=$1; ALT=$2; shift; shift
python -m paper_2007_16122_b200.build > /dev/null
for i in 1 2; do
  for v in main alt; do
    if [ $v = alt ]; then export COLD_LIB_AB=$PWD/$ALT; else unset COLD_LIB_AB; fi
    timeout 300 python bench.py --no-latency --no-e2e --no-cpu --steps 5 "$@" > gpurun_out/ab_${TAG}_$v$i.jsonl 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_$v$i.jsonl').read().splitlines()[-1]);k=d['kernels']
print('$v', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"
  done
done
unset COLD_LIB_AB
