# in-core pivoted LDL / LU schedule variants: parity, then timing (B2D_REST_KCHUNK, B2D_LDL_SPLIT)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "in_core_equals_block_walk or ldl or lu" 2>&1 | tail -2
for sp in ${SPLITS:-0 1}; do for kc in ${KCS:-8}; do echo "KC=$kc SPLIT=$sp"; B2D_LDL_SPLIT=$sp B2D_REST_KCHUNK=$kc python tools/ldl_bench.py --steps 2 2>&1 | grep memdet_ldl | tail -1; done; done
B2D_LDL_TRACE=1 python tools/ldl_bench.py --steps 2 2>&1 | tail -48
