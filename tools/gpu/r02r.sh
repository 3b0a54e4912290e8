# the N > 1 bench path on one GPU (gloo, both ranks on cuda:0): a path check, not a bench number
set -x
python -m paper_2007_16122_b200.build > /dev/null
COLD_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --requests 256 --ads 10000 --steps 3 --warmup 3 --no-cpu --latency-requests 200 > gpurun_out/bench_n2_onegpu_r02r.jsonl 2> gpurun_out/bench_n2_onegpu_r02r.err; echo n2 rc=$?
tail -c 2500 gpurun_out/bench_n2_onegpu_r02r.jsonl; tail -5 gpurun_out/bench_n2_onegpu_r02r.err
COLD_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 3 --requests 100 --ads 3000 --steps 2 --warmup 3 --no-cpu --latency-requests 100 > gpurun_out/bench_n3_onegpu_r02r.jsonl 2> gpurun_out/bench_n3_onegpu_r02r.err; echo n3 rc=$?
tail -c 1200 gpurun_out/bench_n3_onegpu_r02r.jsonl; tail -5 gpurun_out/bench_n3_onegpu_r02r.err
