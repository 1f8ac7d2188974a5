#!/bin/bash
out=gpurun_out/grp_ab2.txt
: > $out
for cfg in "B2D_LDL_GROUPS=4 B2D_REST_KCHUNK=32 B2D_LDL_FRONT_UE=8" "B2D_LDL_GROUPS=4 B2D_REST_KCHUNK=24" "B2D_LDL_GROUPS=0 B2D_REST_KCHUNK=32"; do
  echo "=== $cfg" >> $out
  env $cfg timeout 600 python tools/ldl_tl.py --tag "$cfg" --out gpurun_out/ldl_tl_tmp.txt 2>&1 | grep -v "ldl trace" >> $out
done
for cfg in "B2D_REST_KCHUNK=16" "B2D_REST_KCHUNK=32" "B2D_LDL_ROWS=1 B2D_LDL_GROUPS=4 B2D_REST_KCHUNK=32" "B2D_LDL_ROWS=1 B2D_LDL_GROUPS=4 B2D_REST_KCHUNK=16"; do
  echo "=== C3-size $cfg" >> $out
  env $cfg timeout 900 python tools/ldl_tl.py --n 65536 --nb 16 --steps 2 --tag "C3 $cfg" --out gpurun_out/ldl_tl_tmp.txt 2>&1 | grep -v "ldl trace" >> $out
done
grep -n "median" $out
