#!/bin/bash
# host-input memdet_cholesky: eager band catch-ups (B2D_EAGER_CATCH) A/B -- pinned (C2 / C3 size)
# and a MEMDET01 file (pageable, staged; tools/file_input_bench.py)
out=gpurun_out/eager_ab2.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "eager or staged_equals_pinned or cholesky" > gpurun_out/eager_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/eager_pytest.log
tail -4 gpurun_out/eager_pytest.log
for e in 0 1; do
  TAG="B2D_EAGER_CATCH=$e" B2D_EAGER_CATCH=$e python tools/e2e_time.py >> $out 2>&1
done
for e in 0 1; do
  echo "=== file input, B2D_EAGER_CATCH=$e" >> $out
  B2D_EAGER_CATCH=$e python tools/file_input_bench.py 2>&1 | grep "cholesky" >> $out
done
cat $out
