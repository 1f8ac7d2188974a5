# C2 device path: outer-panel width / tail sweep (after the left-looking below-panel change)
run() { echo "== $*"; env "$@" python tools/one_step.py --steps 4 | tail -1; }
run B2D_X=0
run B2D_TAIL_W=4
run B2D_TAIL_W=16
run B2D_TAIL_TILES=32
run B2D_TAIL_TILES=96
run B2D_PANEL_TILES=12
run B2D_PANEL_TILES=20
run B2D_PANEL_TILES=24
run B2D_X=0
