mkdir -p gpurun_out
SP_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g131_b4.log 2>&1; echo "exit $?" >> gpurun_out/g131_b4.log
SP_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/g131_ref2.log 2>&1; echo "exit $?" >> gpurun_out/g131_ref2.log
