set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:forest_build -c 1 -f -o gpurun_out/r2r_forest python tools/forest_once.py cfg2 > gpurun_out/r2r_ncu.log 2>&1
tail -3 gpurun_out/r2r_ncu.log
