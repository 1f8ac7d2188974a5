# round-2 ncu --set full captures (one GPU): the top kernel of the C2 Cholesky step (first trailing
# "rest" Schur update) and the pivoted-LDL panel / bulk kernels (4096 block, tools/ldl_prof).
mkdir -p gpurun_out/ncu
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
$N -k 'regex:gemm_kernel<\(int\)0>' -s 32 -c 1 -o gpurun_out/ncu/r02_gemm -f python tools/one_step.py --n 32768 > gpurun_out/ncu/r02_gemm.log 2>&1
$N -k regex:ldl_bulk_kernel -s 2 -c 1 -o gpurun_out/ncu/r02_bulk -f ./tools/ldl_prof 4096 > gpurun_out/ncu/r02_bulk.log 2>&1
$N -k regex:ldl_panel_cluster_kernel -s 4 -c 1 -o gpurun_out/ncu/r02_panel -f ./tools/ldl_prof 4096 > gpurun_out/ncu/r02_panel.log 2>&1
ncu -i gpurun_out/ncu/r02_gemm.ncu-rep --page raw --csv > gpurun_out/ncu/r02_gemm_raw.csv 2>&1
for r in r02_bulk r02_panel r02_gemm; do python tools/ncu_kernel_summary.py gpurun_out/ncu/$r.ncu-rep > gpurun_out/ncu/$r.json 2>&1; done
ls -la gpurun_out/ncu
