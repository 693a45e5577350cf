mkdir -p gpurun_out
(timeout 300 python tools/gemm_sweep.py 512 768 1024) > gpurun_out/g117.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/g117_bench.log 2>&1
SP_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --no-decode --no-cpu-baseline > gpurun_out/g117_b2.log 2>&1
