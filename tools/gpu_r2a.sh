set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"join_kernel|replay_kernel" -c 5 -o gpurun_out/r2a_join python tools/profile_build.py --iters 2 > gpurun_out/r2a_ncu_join.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a_launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --e2e-steps 1 > gpurun_out/r2a_ncu_bench.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python __graft_entry__.py > gpurun_out/r2a_sanitizer_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/r2a_sanitizer_summary.txt
done
cat gpurun_out/r2a_sanitizer_summary.txt
