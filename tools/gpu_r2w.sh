set -x
mkdir -p gpurun_out
for mode in 1 0; do
ANNK_L2_PERSIST=$mode timeout 600 python bench.py --skip-cpu --skip-cfg4 > gpurun_out/r2w_bench_l2_$mode.json 2> gpurun_out/r2w_bench_l2_$mode.err; echo "rc=$?"
done
python - <<'PY'
import json
for m in (1,0):
    d=json.loads(open(f'gpurun_out/r2w_bench_l2_{m}.json').read().strip().splitlines()[-1])
    print('L2_PERSIST',m,'value',d['value'],'e2e',d['e2e']['value'],'qps',d['search_qps_at_recall_0.9'], 'search_ms', d['search_kernels_ms'])
    print('   ', {k:round(v/5,2) for k,v in list(d['kernels_ms'].items())[:6]})
PY
