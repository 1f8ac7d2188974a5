#!/bin/bash
# host-ingest (e2e) path knob sweep at C2
run() { echo "== $*"; env "$@" python tools/one_step.py --steps 3 --host | tail -1; }
run B2D_X=0
run B2D_HEAD_TILES=16 B2D_HEAD_W=4
run B2D_HEAD_TILES=16 B2D_HEAD_W=8
run B2D_HEAD_TILES=32 B2D_HEAD_W=8
run B2D_COL_LAT_US=300
run B2D_COL_LAT_US=150
run B2D_COL_LAT_US=300 B2D_HEAD_TILES=16 B2D_HEAD_W=8
run B2D_COL_LAT_US=2000
run B2D_COL_LAT_US=300 B2D_HEAD_TILES=32 B2D_HEAD_W=4
