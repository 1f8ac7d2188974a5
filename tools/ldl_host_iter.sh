# pivoted LDL in core from host memory: parity, then C2 pinned / file timings
timeout 900 python -m pytest tests -m gpu -q -x -k "ldl or file_input" 2>&1 | tail -2
timeout 300 python tools/file_input_bench.py 2>&1 | grep -E 'ldl' | sed -n '2p;4p'
