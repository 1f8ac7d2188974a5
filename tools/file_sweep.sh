# MEMDET01-file (pageable) input: staging-rate model sweep (band plan)
for g in 14 25 35 50; do echo "STAGE_GBS=$g"; B2D_STAGE_GBS=$g timeout 300 python tools/file_input_bench.py 2>&1 | grep -E 'from MEMDET01' | sed -n '2p;4p'; done
