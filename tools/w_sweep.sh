#!/bin/bash
python tools/one_step.py --n 32768 --steps 2 | tail -1 | sed 's/^/base /'
for t in 32 64; do B2D_TAIL_TILES=$t python tools/one_step.py --n 32768 --steps 2 | tail -1 | sed "s/^/tail=$t /"; done
python tools/one_step.py --n 32768 --steps 2 --host | tail -1 | sed 's/^/host base /'
for h in 16 32 64; do B2D_HEAD_TILES=$h python tools/one_step.py --n 32768 --steps 2 --host | tail -1 | sed "s/^/host head=$h /"; done
timeout 900 python -m pytest tests -m gpu -x -q -k "golden or ragged or out_of_core or device_tensor" 2>&1 | tail -1
