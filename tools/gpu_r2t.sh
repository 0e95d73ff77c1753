set -x
mkdir -p gpurun_out
python -c "
import paper_1609_07228_b200 as A
for g in (2000, 20000, 100000): print('i8 peak groups', g, A.measure_i8_peak(g), 'TOP/s')
" 2>&1 | tail -4
timeout 600 python bench.py --skip-cpu > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2t_bench.err
