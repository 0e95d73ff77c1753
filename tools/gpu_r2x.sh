set -x
mkdir -p gpurun_out
for gb in 32 64; do
ANNK_OFFER_GB=$gb timeout 600 python bench.py --skip-cpu --skip-cfg4 --e2e-steps 1 > gpurun_out/r2x_bench_gb$gb.json 2> gpurun_out/r2x_bench_gb$gb.err; echo "rc=$?"
done
python - <<'PY'
import json
for m in (32,64):
    d=json.loads(open(f'gpurun_out/r2x_bench_gb{m}.json').read().strip().splitlines()[-1])
    print('OFFER_GB',m,'value',d['value'],'e2e',d['e2e']['value'],'qps',d['search_qps_at_recall_0.9'])
    print('   ', {k:round(v/5,2) for k,v in d['kernels_ms'].items()})
PY
