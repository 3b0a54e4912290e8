set -x
python -m paper_2007_16122_b200.build > /dev/null
COLD_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --requests 1024 --no-serve > gpurun_out/bench_n2_onegpu_r03bb.jsonl 2> gpurun_out/bench_n2_onegpu_r03bb.err; echo n2 rc=$?
tail -c 1500 gpurun_out/bench_n2_onegpu_r03bb.jsonl
