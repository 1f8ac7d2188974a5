# pivoted LDL: parity, then the in-core schedule knobs at C2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ldl" 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 120 python tools/ldl_bench.py --steps 3 2>&1 | grep memdet_ldl | tail -1; }
run B2D_X=0
run B2D_REST_KCHUNK=0
run B2D_LDL_SPLIT=0
run B2D_LDL_SCHED=1
run B2D_LDL_PERSIST=1
