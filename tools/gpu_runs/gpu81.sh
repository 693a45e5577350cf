mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g81t.log 2>&1; echo "exit $?" >> gpurun_out/g81t.log
SP_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --decode-batch 8 > gpurun_out/g81_b2.log 2>&1; echo "exit $?" >> gpurun_out/g81_b2.log
