# out-of-core Cholesky walk: parity, then timing with / without the diagonal look-ahead
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "out_of_core or ooc" 2>&1 | tail -2
python tools/ooc_bench.py --n 65536 --nb 4 --budget-gb 24 2>&1 | tail -4
B2D_OOC_NO_LOOKAHEAD=1 python tools/ooc_bench.py --n 65536 --nb 4 --budget-gb 24 --skip-incore 2>&1 | tail -2
python tools/ooc_bench.py --n 65536 --nb 8 --budget-gb 24 --skip-incore 2>&1 | tail -2
