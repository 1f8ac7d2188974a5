run() { echo "== $*"; env "$@" timeout 300 python tools/ldl_dev.py --cfg C2 2>&1 | tail -1; }
run B2D_X=0
run B2D_REST_KCHUNK=4
run B2D_REST_KCHUNK=2
run B2D_REST_KCHUNK=1
run B2D_LDL_PERSIST=1
B2D_LDL_TRACE=1 timeout 300 python tools/ldl_dev.py --cfg C2 --steps 1 2>&1 | tail -60
