set -x
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --comm gloo --steps 2 --warmup 3 > gpurun_out/r2v_bench_gpus2_gloo.json 2> gpurun_out/r2v_bench_gpus2_gloo.err; echo "gpus2 rc=$?"
tail -2 gpurun_out/r2v_bench_gpus2_gloo.err
make debug > gpurun_out/r2v_make_debug.log 2>&1; echo "make debug rc=$?"
bash tools/gpu_checked_tests.sh > /dev/null 2>&1
tail -6 gpurun_out/checked_tests.log
