# generic LU in core: parity, then n = 32768 timing (device-resident, then through memdet_lu from pinned host memory)
timeout 900 python -m pytest tests -m gpu -q -x -k "lu or acceptance" 2>&1 | tail -2
python tools/lu_bench.py --steps 2 2>&1 | tail -1
python tools/lu_bench.py --steps 2 2>&1 | grep -E 'memdet_lu n=' | tail -1
