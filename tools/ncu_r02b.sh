#!/bin/bash
# round-2 final: ncu --set full of the top kernel (first trailing "rest" Schur update of the C2
# Cholesky step) at HEAD, then the ncu launch list of the bench command (after its plain run).
mkdir -p gpurun_out/ncu
python tools/one_step.py --n 32768 > gpurun_out/ncu/r02b_plain.log 2>&1 || exit 1
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
$N -k 'regex:gemm_kernel<\(int\)0>' -s 32 -c 1 -o gpurun_out/ncu/r02b_gemm -f python tools/one_step.py --n 32768 > gpurun_out/ncu/r02b_gemm.log 2>&1
ncu -i gpurun_out/ncu/r02b_gemm.ncu-rep --page raw --csv > gpurun_out/ncu/r02b_gemm_raw.csv 2>&1
python tools/ncu_kernel_summary.py gpurun_out/ncu/r02b_gemm.ncu-rep > gpurun_out/ncu/r02b_gemm.json 2>&1
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ozaki --no-ooc --no-c3 --no-file > gpurun_out/r02b_bench_plain.json 2> gpurun_out/r02b_bench_plain.err || exit 2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r02b_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ozaki --no-ooc --no-c3 --no-file \
    > gpurun_out/r02b_ncu_bench.log 2>&1
echo "ncu exit $?" >> gpurun_out/r02b_ncu_bench.log
ls -la gpurun_out/ncu gpurun_out/r02b*
