# round-2 final evidence: bench lines (cfg2 with CPU baseline, cfg1, cfg3, cfg5), the ncu launch
# list of the bench command, full captures of the exact-kNN kernels and the forest kernel
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2u_bench_cfg2.json 2> gpurun_out/r2u_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config cfg5 --skip-cpu --skip-cfg4 --steps 2 --warmup 3 > gpurun_out/r2u_bench_cfg5.json 2> gpurun_out/r2u_bench_cfg5.err; echo "cfg5 rc=$?"
timeout 1200 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/r2u_bench_cfg3.json 2> gpurun_out/r2u_bench_cfg3.err; echo "cfg3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2u_launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 1 > gpurun_out/r2u_ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bf_tc_u8_kernel|bf_merge_kernel|home_kernel|prune_kernel" -c 12 -f -o gpurun_out/r2u_bf python tools/prof_bf_once.py 1000000 > gpurun_out/r2u_ncu_bf.log 2>&1; echo "bf rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:forest_build -c 1 -f -o gpurun_out/r2u_forest python tools/forest_once.py cfg2 > gpurun_out/r2u_ncu_forest.log 2>&1; echo "forest rc=$?"
ls -la gpurun_out | tail -12
