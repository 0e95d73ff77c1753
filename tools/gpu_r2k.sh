set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
python bench.py --config cfg5 --skip-cpu --skip-cfg4 --steps 2 --warmup 3 > gpurun_out/r2k_bench_cfg5.json 2> gpurun_out/r2k_bench_cfg5.err
python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/r2k_bench_cfg3.json 2> gpurun_out/r2k_bench_cfg3.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 1 > gpurun_out/r2k_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"join_kernel|replay_kernel|offer_compact|init_kernel" -c 6 -o gpurun_out/r2k_build python tools/profile_build.py --iters 2 > gpurun_out/r2k_ncu_build.log 2>&1
echo done
