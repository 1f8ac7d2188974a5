#!/bin/bash
# quick GPU iteration: C2 timing at panel widths, launch list at n=16384, then gpu tests
for w in ${WIDTHS:-4 8}; do B2D_PANEL_TILES=$w python tools/one_step.py --n ${N:-32768} --steps 3 | tail -1; done
B2D_PANEL_TILES=8 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv python tools/one_step.py --n 16384 > gpurun_out/ncu_iter.log 2>&1
python tools/launch_summary.py gpurun_out/launches_iter.csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
