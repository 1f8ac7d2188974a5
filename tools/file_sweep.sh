# MEMDET01-file (pageable) input: staging-rate model sweep, then the file-input bench
for g in 14 10 20; do echo "STAGE_GBS=$g"; B2D_STAGE_GBS=$g timeout 300 python tools/file_input_bench.py 2>&1 | grep -E 'cholesky from MEMDET01' | tail -1; done
echo "no staging"; B2D_HOST_STAGING=0 timeout 300 python tools/file_input_bench.py 2>&1 | grep -E 'from MEMDET01' | tail -3
