#!/bin/bash
# One gpurun call: GPU tests, smoke, the default bench line, then the ncu launch list of the
# same bench command (cold, serialised; only after the plain run exited 0).
#   gpurun --timeout 3600 -- bash tools/gpu_round.sh [tag]
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
nvidia-smi > $out/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1
echo "smoke exit $?" >> $out/${tag}_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $out/${tag}_pytest_gpu.log
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
rc=$?
echo "bench exit $rc" >> $out/${tag}_bench.err
if [ $rc -eq 0 ] && [ "${NO_NCU:-0}" != 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ozaki --no-ooc --no-c3 --no-file \
    > $out/${tag}_ncu_bench.log 2>&1
  echo "ncu exit $?" >> $out/${tag}_ncu_bench.log
fi
