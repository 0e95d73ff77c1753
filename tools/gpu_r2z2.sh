set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_sharded.py -m gpu -x -q > gpurun_out/r2z_tests.log 2>&1; echo "rc=$?"
tail -4 gpurun_out/r2z_tests.log
for c in cfg2 cfg3 cfg5; do
timeout 900 python bench.py --config $c --skip-cpu --skip-cfg4 --e2e-steps 1 --steps 2 --warmup 3 > gpurun_out/r2z_bench_$c.json 2> gpurun_out/r2z_bench_$c.err; echo "rc=$?"
done
python - <<'PY'
import json
for c in ('cfg2','cfg3','cfg5'):
    d=json.loads(open(f'gpurun_out/r2z_bench_{c}.json').read().strip().splitlines()[-1])
    print(c,'value',d['value'],'e2e',d['e2e']['value'])
    print('   ', {k:round(v/2,2) for k,v in d['kernels_ms'].items() if 'rev' in k or 'sort' in k})
PY
