set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 1 > gpurun_out/r2h_ncu_bench.log 2>&1; echo "launch list rc=$?"
python tools/launch_shares.py gpurun_out/r2h_launches.csv > gpurun_out/r2h_launch_shares.txt; head -20 gpurun_out/r2h_launch_shares.txt
