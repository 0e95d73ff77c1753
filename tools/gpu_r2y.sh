set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_config_parity.py -m gpu -x -q --durations=5 > gpurun_out/r2y_tests.log 2>&1; echo "rc=$?"
tail -15 gpurun_out/r2y_tests.log
