for v in s4_p1 s3_p4 s2_p4; do
  for cfg in C2; do
    B2D_LIB_OVERRIDE=tools/varlib/lib_$v.so timeout 300 python tools/ldl_dev.py --cfg $cfg 2>&1 | tail -1 | sed "s/^/$v /"
    B2D_LIB_OVERRIDE=tools/varlib/lib_$v.so timeout 300 python tools/ldl_dev.py --cfg $cfg --chol 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
B2D_LIB_OVERRIDE=tools/varlib/lib_s2_p4.so B2D_LDL_TRACE=1 timeout 300 python tools/ldl_dev.py --cfg C2 --steps 1 2>&1 | grep "factor-\|next-col" | tail -24
