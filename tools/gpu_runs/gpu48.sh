mkdir -p gpurun_out
SP_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --decode-batch 8 > gpurun_out/g48_b2.log 2>&1; echo "exit $?" >> gpurun_out/g48_b2.log
SP_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/g48_r2.log 2>&1; echo "exit $?" >> gpurun_out/g48_r2.log
