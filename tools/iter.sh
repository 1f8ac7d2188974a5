#!/bin/bash
# quick GPU iteration: C2 timing (device + host-ingest paths), gpu tests
for w in ${WIDTHS:-8}; do B2D_PANEL_TILES=$w python tools/one_step.py --n ${N:-32768} --steps 3 | tail -1; done
python tools/one_step.py --n ${N:-32768} --steps 3 --host | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
