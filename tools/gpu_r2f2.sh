set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or refine_and_finalize or piecewise" > gpurun_out/r2f2_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r2f2_tests.log
timeout 900 python bench.py --skip-cpu --skip-cfg4 --steps 3 --warmup 3 --e2e-steps 3 > gpurun_out/r2f2_bench.json 2> gpurun_out/r2f2_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2f2_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2f2_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e'],'e2e_fb',d['e2e_with_forest_build']['value'])
PY
