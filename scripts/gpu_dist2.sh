mkdir -p gpurun_out
MLSB_BENCH_DIST=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?
tail -c 1500 gpurun_out/bench2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo rc=$?
tail -c 600 gpurun_out/ref2.json
