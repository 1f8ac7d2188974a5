#!/bin/bash
# e2e (pinned host ingest) sweep over the band-plan model parameters
for lat in 900 600 300; do
  for bw in 48 55; do
    r=$(B2D_COL_LAT_US=$lat B2D_PCIE_GBS=$bw python tools/one_step.py --host --steps 3 | tail -1 | awk '{print $3}')
    echo "col_lat=$lat pcie=$bw -> $r ms"
  done
done
