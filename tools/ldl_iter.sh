# pivoted LDL quick iteration: kernel-level profile, parity, C2 timing
./tools/ldl_prof 4096 2>&1 | grep -E 'panel|one-launch|bulk' | head -4
timeout 900 python -m pytest tests -m gpu -q -x -k "ldl" 2>&1 | tail -2
python tools/ldl_bench.py --steps 3 2>&1 | grep memdet_ldl | tail -1
