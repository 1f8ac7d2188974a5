run() { echo "== $*"; env "$@" timeout 300 python tools/ldl_dev.py --cfg C2 2>&1 | tail -1; }
run B2D_LDL_URGENT=0
run B2D_X=0
run B2D_LDL_COL_STREAMS=2
run B2D_LDL_COL_STREAMS=16
timeout 300 python tools/ldl_dev.py --cfg C3 --steps 2 2>&1 | tail -1
B2D_LDL_URGENT=0 timeout 300 python tools/ldl_dev.py --cfg C3 --steps 2 2>&1 | tail -1
B2D_LDL_TRACE=1 timeout 300 python tools/ldl_dev.py --cfg C2 --steps 1 2>&1 | tail -70 | grep -v "^\[ldl trace\].*" | head -2
B2D_LDL_TRACE=1 timeout 300 python tools/ldl_dev.py --cfg C2 --steps 1 2>&1 | tail -75 | head -72
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ldl" 2>&1 | tail -2
