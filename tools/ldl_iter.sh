# pivoted LDL quick iteration: parity subset, C2 timing + trace
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ldl" 2>&1 | tail -2
python tools/ldl_bench.py --steps 3 2>&1 | grep memdet_ldl | tail -1
B2D_LDL_TRACE=1 python tools/ldl_bench.py --steps 2 2>&1 | grep -E 'factor-(begin|end)|end 8' | tail -17
