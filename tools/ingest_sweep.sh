# pinned host input: strips enqueued all up front (0) or band by band with the factorisation (1)
for pr in 0 1 0 1; do echo "PROGRESSIVE=$pr"; B2D_INGEST_PROGRESSIVE=$pr python tools/one_step.py --host --steps 3 | tail -1; done
for pr in 0 1; do echo "PROGRESSIVE=$pr"; B2D_INGEST_PROGRESSIVE=$pr python tools/ldl_bench.py --steps 2 2>&1 | grep memdet_ldl | tail -1; done
