#!/bin/bash
# ORACLE — TEST INFRASTRUCTURE ONLY.  Compiles the reference's own native LDL kernel
# (/root/reference/pkg/src/oocdet/kernels/_ldl.pyx, Cython) where it lies, into oracle/_ref/,
# so tests can check the C restatement (oracle/ldl_tile.c) against it.  Nothing is copied into
# the repository: outputs go to the git-ignored oracle/_ref/ only.
set -e
SRC=/root/reference/pkg/src/oocdet/kernels/_ldl.pyx
OUT="$(cd "$(dirname "$0")" && pwd)/_ref"
[ -f "$SRC" ] || { echo "reference not mounted; skipping oracle/_ref"; exit 0; }
mkdir -p "$OUT"
python -m cython -3 "$SRC" -o "$OUT/_ldl.c" >/dev/null
PYINC=$(python -c "import sysconfig; print(sysconfig.get_paths()['include'])")
EXT=$(python -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
gcc -O2 -fPIC -shared -I"$PYINC" "$OUT/_ldl.c" -o "$OUT/_ldl$EXT"
echo "$OUT/_ldl$EXT"
