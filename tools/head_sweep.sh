#!/bin/bash
# device-path head/tail panel-width sweep at C2, each config twice, 5 steps
run() { echo "== $*"; env "$@" python tools/one_step.py --steps 5 | tail -1; }
for rep in 1 2; do
run B2D_X=0
run B2D_DEV_HEAD_TILES=8 B2D_HEAD_W=8
run B2D_DEV_HEAD_TILES=16 B2D_HEAD_W=8
run B2D_DEV_HEAD_TILES=4 B2D_HEAD_W=4
run B2D_DEV_HEAD_TILES=8 B2D_HEAD_W=4
done
