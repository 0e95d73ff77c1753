set -x
mkdir -p gpurun_out
ANNK_LIB=paper_1609_07228_b200/libannkit_ft.so timeout 300 python tools/time_forest.py cfg2 > gpurun_out/r2p_forest_timing.log 2>&1
timeout 600 python bench.py --skip-cpu > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo "bench rc=$?"
tail -30 gpurun_out/r2p_forest_timing.log
