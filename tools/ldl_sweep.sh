#!/bin/bash
# A/B sweep of in-core memdet_ldl switches at C2 (and optionally C3) in one gpurun call:
#   gpurun -- bash tools/ldl_sweep.sh "B2D_LDL_LA=0" "B2D_LDL_LA=4" ...
# each argument is an environment assignment list (space separated) for one tools/ldl_tl.py run.
out=gpurun_out
mkdir -p $out
for cfg in "$@"; do
  echo "=== $cfg" >> $out/ldl_sweep.log
  env $cfg timeout 600 python tools/ldl_tl.py --out $out/ldl_tl_tmp.txt --tag "$cfg" ${LDL_ARGS} >> $out/ldl_sweep.log 2>&1
done
