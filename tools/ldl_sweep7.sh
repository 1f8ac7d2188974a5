for env in "B2D_X=0" "CUDA_DEVICE_MAX_CONNECTIONS=32" "B2D_LDL_COL_STREAMS=1" "CUDA_DEVICE_MAX_CONNECTIONS=32 B2D_LDL_COL_STREAMS=2"; do
  echo "== $env"
  env $env B2D_LDL_TRACE=1 timeout 300 python tools/ldl_dev.py --cfg C2 --steps 1 2>&1 | grep "factor-begin 2\|next-col-end 1\|factor-begin 4\|next-col-end 3\|C2 ldl"
  env $env timeout 300 python tools/ldl_dev.py --cfg C2 --steps 3 2>&1 | tail -1
done
