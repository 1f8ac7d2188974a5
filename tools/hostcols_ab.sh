#!/bin/bash
out=gpurun_out/hostcols_ab.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "pivoted_ldl_in_core or group_pipeline or staged_equals_pinned" > gpurun_out/hostcols_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/hostcols_pytest.log
tail -3 gpurun_out/hostcols_pytest.log
for r in 1 2; do for e in 0 1; do
  FN=ldl TAG="B2D_LDL_HOST_COLS=$e" B2D_LDL_HOST_COLS=$e python tools/e2e_time.py >> $out 2>&1
done; done
for e in 0 1; do
  FN=ldl NB=16 TAG="C3-size B2D_LDL_HOST_COLS=$e" B2D_LDL_HOST_COLS=$e python tools/e2e_time.py 65536 >> $out 2>&1
done
cat $out
