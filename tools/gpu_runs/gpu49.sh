mkdir -p gpurun_out
timeout 600 python tools/host_profile.py 1 2048 32 > gpurun_out/g49_b1.log 2>&1
timeout 600 python tools/host_profile.py 64 2048 32 > gpurun_out/g49_b64.log 2>&1
