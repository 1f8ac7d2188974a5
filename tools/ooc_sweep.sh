#!/bin/bash
# out-of-core (n=65536, 4 blocks, 24 GB budget) vs panel schedule of the diagonal-block factorisation
run() { echo "== $*"; env "$@" python tools/ooc_bench.py --n 65536 --nb 4 --budget-gb 24 --skip-incore --steps 2 2>&1 | grep "out-of-core" | tail -1; }
run B2D_X=0
run B2D_PANEL_TILES=8
run B2D_PANEL_TILES=8 B2D_TAIL_TILES=32 B2D_TAIL_W=4
run B2D_TAIL_TILES=32
for n in 16384; do
  echo "== in-core n=$n"; python tools/one_step.py --n $n --steps 3 | tail -1
  B2D_PANEL_TILES=8 python tools/one_step.py --n $n --steps 3 | tail -1
  B2D_PANEL_TILES=8 B2D_TAIL_TILES=32 B2D_TAIL_W=4 python tools/one_step.py --n $n --steps 3 | tail -1
done
