#!/bin/bash
# C2 device + host paths, C3-size device path, OOC at n=32768 forced, gpu tests
python tools/one_step.py --steps 3 | tail -1
python tools/one_step.py --steps 3 --host | tail -1
for w in ${HOSTW:-}; do B2D_PANEL_TILES=$w python tools/one_step.py --steps 3 --host | tail -1; done
python tools/one_step.py --n 65536 --steps 2 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
