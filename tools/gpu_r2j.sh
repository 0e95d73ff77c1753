set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py tests/test_gpu_config_parity.py -m gpu -x -q > gpurun_out/r2m2_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2m2_tests.log
timeout 900 python bench.py --skip-cpu --skip-cfg4 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/r2m2_bench_cfg2.json 2> gpurun_out/r2m2_bench_cfg2.err; echo "cfg2 rc=$?"
ANNK_TRACE=1 timeout 900 python bench.py --config cfg5 --skip-cpu --skip-cfg4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/r2m2_bench_cfg5.json 2> gpurun_out/r2m2_bench_cfg5.err; echo "cfg5 rc=$?"
grep "join \[" gpurun_out/r2m2_bench_cfg5.err | tail -10
python - <<'PY'
import json
for c in ('cfg2','cfg5'):
    d=json.loads(open(f'gpurun_out/r2m2_bench_{c}.json').read().strip().splitlines()[-1])
    print(c,'value',d['value'],'e2e',d['e2e']['value'])
    print(sorted(((round(v/d['steps'],1),k) for k,v in d['kernels_ms'].items()),reverse=True)[:5])
PY
