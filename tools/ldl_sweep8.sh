B2D_LDL_PERSIST=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ldl" 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 300 python tools/ldl_dev.py --cfg C2 2>&1 | tail -1; }
run B2D_X=0
run B2D_LDL_PERSIST=1
run B2D_LDL_PERSIST=2
run B2D_LDL_PERSIST=1 CUDA_DEVICE_MAX_CONNECTIONS=32
B2D_LDL_PERSIST=1 timeout 300 python tools/ldl_dev.py --cfg C3 --steps 2 2>&1 | tail -1
B2D_LDL_PERSIST=1 B2D_LDL_TRACE=1 timeout 300 python tools/ldl_dev.py --cfg C2 --steps 1 2>&1 | grep "factor-\|next-col" | tail -24
