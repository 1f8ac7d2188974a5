#!/bin/bash
for n in 32768 65536; do for l in -1 1 2 4 8; do B2D_LAZY_STEPS=$l python tools/one_step.py --n $n --steps 2 | tail -1 | sed "s/^/lazy=$l /"; done; done
