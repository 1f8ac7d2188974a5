# pivoted LDL schedule knobs at C2
run() { echo "== $*"; env "$@" python tools/ldl_bench.py --steps 3 2>&1 | grep memdet_ldl | tail -1; }
run B2D_X=0
run B2D_REST_KCHUNK=4
run B2D_REST_KCHUNK=2
run B2D_LDL_PERSIST=1
run B2D_LDL_PERSIST=1 B2D_REST_KCHUNK=32
run B2D_LDL_SCHED=1
