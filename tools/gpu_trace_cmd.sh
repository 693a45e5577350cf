set -e
SP_NVCC_EXTRA=-DSTEP_TRACE python -m paper_2507_11830_b200.build --force > /dev/null
cp paper_2507_11830_b200/libshiftpar.so paper_2507_11830_b200/libshiftpar_trace.so
python -m paper_2507_11830_b200.build --force > /dev/null
mkdir -p gpurun_out
timeout 300 python tools/step_trace.py 1 2048 --layers 2 --ctas > gpurun_out/trace_b1.txt 2>&1
timeout 300 python tools/step_trace.py 64 2048 --layers 2 --ctas > gpurun_out/trace_b64.txt 2>&1
