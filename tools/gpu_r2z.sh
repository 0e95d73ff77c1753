set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_sharded.py -m gpu -x -q > gpurun_out/r2z_tests.log 2>&1; echo "rc=$?"
tail -4 gpurun_out/r2z_tests.log
timeout 600 python bench.py --skip-cpu --skip-cfg4 --e2e-steps 1 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo "rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2z_bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],'qps',d['search_qps_at_recall_0.9'])
print('   ', {k:round(v/5,2) for k,v in d['kernels_ms'].items()})
PY
