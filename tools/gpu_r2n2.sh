set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n2_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2n2_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n2_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/r2n2_smoke.log
