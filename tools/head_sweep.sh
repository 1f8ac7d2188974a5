#!/bin/bash
# e2e (pinned host ingest) head-panel sweep at C2
run() { echo "== $*"; env "$@" python tools/one_step.py --host --steps 3 | tail -1; }
run B2D_X=0
run B2D_HEAD_TILES=8 B2D_HEAD_W=4
run B2D_HEAD_TILES=16 B2D_HEAD_W=4
run B2D_HEAD_TILES=16 B2D_HEAD_W=8
run B2D_HEAD_TILES=32 B2D_HEAD_W=8
run B2D_HEAD_TILES=4 B2D_HEAD_W=4
