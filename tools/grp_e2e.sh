#!/bin/bash
# memdet_ldl end to end from pinned host memory: group pipeline switches A/B (C2; C3-sized with NB=16)
out=gpurun_out/grp_e2e.txt
: > $out
for cfg in "B2D_LDL_GROUPS=0 B2D_REST_KCHUNK=16" "B2D_LDL_GROUPS=0" "B2D_LDL_GROUPS=4" "B2D_LDL_GROUPS=4 B2D_LDL_FRONT=0" "B2D_LDL_GROUPS=4 B2D_LDL_FRONT=0 B2D_REST_KCHUNK=16" "B2D_LDL_GROUPS=4 B2D_REST_KCHUNK=16" "B2D_LDL_GROUPS=4 B2D_LDL_FRONT_UE=8"; do
  env FN=ldl TAG="$cfg" $cfg timeout 600 python tools/e2e_time.py >> $out 2>&1
done
for cfg in "B2D_LDL_ROWS=0 B2D_REST_KCHUNK=16" "B2D_LDL_GROUPS=4" "B2D_LDL_GROUPS=4 B2D_LDL_FRONT=0"; do
  env FN=ldl NB=16 TAG="C3-size $cfg" $cfg timeout 900 python tools/e2e_time.py 65536 >> $out 2>&1
done
cat $out
