for t in $(python - <<'P'
import re
src=open('tests/test_engine_gpu.py').read()
print(' '.join(re.findall(r'^def (test_\w+)', src, re.M)))
P
); do
  timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -k "$t" --tb=short > gpurun_out/et_$t.log 2>&1; echo "$t exit $?" >> gpurun_out/et_summary.log
done
