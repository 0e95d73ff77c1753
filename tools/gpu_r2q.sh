set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "forest or init" > gpurun_out/r2q_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2q_tests.log
timeout 300 python tools/time_forest.py cfg2 2>&1 | tail -4
