set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2f_tests.log
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/r2f_smoke.log
make debug > gpurun_out/r2f_make_debug.log 2>&1; echo "make debug rc=$?"
bash tools/gpu_checked_tests.sh > /dev/null 2>&1
tail -5 gpurun_out/checked_tests.log
