# A/B of a chain-kernel build define: bash tools/gpu/ab_chain.sh <tag> -DDEFINE ...
set -x
TAG=$1; shift
python -m paper_2007_16122_b200.build > /dev/null
bash tools/ab_build.sh alt "$@" > /dev/null 2>&1; echo ab rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or paper_stack or variants or one_wide or prelu or many_small" > gpurun_out/ab_${TAG}_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/ab_${TAG}_tests.log
for i in 1 2; do
  for v in main alt; do
    if [ $v = alt ]; then export COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/alt.so; else unset COLD_LIB_AB; fi
    timeout 300 python bench.py --no-latency --no-e2e --no-cpu --steps 5 > gpurun_out/ab_${TAG}_$v$i.jsonl 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_$v$i.jsonl').read().splitlines()[-1]);k=d['kernels']
print('$v', round(d['value']/1e6,1), {n: round(x['avg_us'],1) for n,x in k.items()}, d['clocks']['sm_mhz'])"
  done
done
unset COLD_LIB_AB
