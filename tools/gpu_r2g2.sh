set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --gpus 2 --comm gloo --steps 2 --warmup 3 > gpurun_out/r2e_bench_cfg2_gloo2.json 2> gpurun_out/r2e_bench_cfg2_gloo2.err; echo "gloo2 rc=$?"
tail -c 1500 gpurun_out/r2e_bench_cfg2_gloo2.json
tail -5 gpurun_out/r2e_bench_cfg2_gloo2.err
