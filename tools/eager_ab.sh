#!/bin/bash
# pinned-host memdet_cholesky: eager band catch-ups (B2D_EAGER_CATCH) A/B at C2 and C3 size
out=gpurun_out/eager_ab.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "eager or staged_equals_pinned or cholesky" > gpurun_out/eager_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/eager_pytest.log
tail -4 gpurun_out/eager_pytest.log
for r in 1 2; do for e in 0 1; do
  TAG="B2D_EAGER_CATCH=$e" B2D_EAGER_CATCH=$e python tools/e2e_time.py >> $out 2>&1
done; done
for e in 0 1; do
  TAG="C3-size B2D_EAGER_CATCH=$e" NB=16 B2D_EAGER_CATCH=$e python tools/e2e_time.py 65536 >> $out 2>&1
done
B2D_EAGER_CATCH=1 python tools/e2e_trace.py 2>&1 | grep "step\|e2e" | grep -v "\-1.00 catch -1.00 rest -1.00" | head -12 >> $out
cat $out
