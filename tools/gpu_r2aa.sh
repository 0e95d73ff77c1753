set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "brute_force" > gpurun_out/r2aa_tests.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r2aa_tests.log
timeout 600 python bench.py --skip-cpu --e2e-steps 1 --steps 2 > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err; echo "rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2aa_bench.json').read().strip().splitlines()[-1])
e=d['exact_knn']; print('exact_knn api',e['seconds_through_api'],'device_ms',e['device_ms'])
PY
