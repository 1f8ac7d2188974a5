# pivoted LDL / LU / OOC quick iteration: parity, C2 LDL timing (left-looking panel solve on / off)
timeout 900 python -m pytest tests -m gpu -q -x -k "ldl or lu or out_of_core or ooc" 2>&1 | tail -2
for lb in 1 0; do echo "LEFT_BELOW=$lb"; B2D_LEFT_BELOW=$lb python tools/ldl_bench.py --steps 3 2>&1 | grep memdet_ldl | tail -1; B2D_LEFT_BELOW=$lb python tools/lu_bench.py --steps 2 2>&1 | tail -1; done
python tools/ooc_bench.py --n 65536 --nb 4 --budget-gb 24 --skip-incore --steps 1 2>&1 | tail -1
