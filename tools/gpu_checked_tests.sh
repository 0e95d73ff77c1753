# The GPU test suite and smoke against the bounds-checked build (make debug:
# -DANNK_DEBUG_CHECKS, every DCHK traps with its file:line) -- this pool has no
# compute-sanitizer, so this is the out-of-bounds evidence.
set -x
mkdir -p gpurun_out
ls -la build/libannkit_b200_dbg.so > gpurun_out/checked_tests.log 2>&1
ANNK_LIB=build/libannkit_b200_dbg.so python -c "import paper_1609_07228_b200 as A, paper_1609_07228_b200._lib as L; print('library:', L.LIB_PATH, A.lib._name)" >> gpurun_out/checked_tests.log 2>&1
ANNK_LIB=build/libannkit_b200_dbg.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider >> gpurun_out/checked_tests.log 2>&1
echo "checked pytest rc=$?" >> gpurun_out/checked_tests.log
ANNK_LIB=build/libannkit_b200_dbg.so python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/checked_tests.log 2>&1
echo "checked smoke rc=$?" >> gpurun_out/checked_tests.log
tail -6 gpurun_out/checked_tests.log
