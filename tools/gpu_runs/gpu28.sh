# full GPU validation of HEAD: tests, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g28_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/g28_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g28_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g28_smoke.log
timeout 600 python bench.py > gpurun_out/g28_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/g28_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g28_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/g28_ref.log
