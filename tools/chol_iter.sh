# in-core Cholesky: parity subset, then C2 device / host timing (B2D_LEFT_BELOW on / off) and a trace
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow and not ldl and not lu" 2>&1 | tail -2
for lb in 1 0; do echo "LEFT_BELOW=$lb"; B2D_LEFT_BELOW=$lb python tools/one_step.py --steps 4 | tail -1; B2D_LEFT_BELOW=$lb python tools/one_step.py --steps 3 --host | tail -1; done
B2D_TRACE=1 python tools/one_step.py --steps 2 2>&1 | grep -E 'step [0-3] |total' | tail -5
