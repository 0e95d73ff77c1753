set -x
mkdir -p gpurun_out
ANNK_DEBUG_FOREST=1 ANNK_LIB=paper_1609_07228_b200/libannkit_ft.so timeout 300 python tools/time_forest.py cfg2 2>&1 | grep -v "phases" | tail -14
ANNK_DEBUG_FOREST=1 timeout 300 python tools/time_forest.py cfg2 2>&1 | tail -12
