set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf_tc.py tests/test_accuracy_vs_k.py -x -q > gpurun_out/r2n_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2n_tests.log
ANNK_BF_STATS=1 timeout 600 python tools/prof_bf.py 1000000 2>&1 | tail -9
ANNK_BF_HOME_CELLS=128 ANNK_BF_STATS=1 timeout 600 python tools/prof_bf.py 1000000 2>&1 | tail -9
ANNK_BF_CELL_ROWS=192 ANNK_BF_HOME_CELLS=96 ANNK_BF_STATS=1 timeout 600 python tools/prof_bf.py 1000000 2>&1 | tail -9
