#!/bin/bash
# A/B of the pivoted LDL group pipeline (B2D_LDL_GROUPS / B2D_LDL_FRONT / B2D_LDL_FRONT_UE): parity
# tests first, then C2 memdet_ldl device step times with the stage trace.
out=gpurun_out/grp_ab.txt
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "pivoted_ldl or ldl" > gpurun_out/grp_ab_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/grp_ab_pytest.log
tail -3 gpurun_out/grp_ab_pytest.log
: > $out
for cfg in "${@:-B2D_LDL_GROUPS=0 B2D_LDL_GROUPS=4}"; do
  echo "=== $cfg" >> $out
  env $cfg timeout 600 python tools/ldl_tl.py --tag "$cfg" --out gpurun_out/ldl_tl_tmp.txt >> $out 2>&1
done
grep -n "median" $out
