#!/bin/bash
run() { echo "== $*"; env "$@" B2D_TRACE=1 python tools/one_step.py --steps 2 2>&1 | grep -E "step 0 |step=1"; }
run B2D_X=0
run B2D_DEV_HEAD_TILES=16 B2D_HEAD_W=8
run B2D_DEV_HEAD_TILES=32 B2D_HEAD_W=8
run B2D_DEV_HEAD_TILES=16 B2D_HEAD_W=4
run B2D_DEV_HEAD_TILES=8 B2D_HEAD_W=4
