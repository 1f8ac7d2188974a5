# ncu --set full captures of the secondary kernels of the C2 Cholesky step (device path):
# the panel TRSM (gemm_kernel<1>), the whole-matrix pack (HBM-bound), the diagonal-tile factor,
# the prefix scan; and the trailing update of the in-core pivoted LDL (K-chunked launch).
set -x
mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on"
$N --kernel-name-base demangled -k 'regex:gemm_kernel<\(int\)1>' -s 20 -c 1 -o gpurun_out/ncu/trsm -f python tools/one_step.py --steps 1 > gpurun_out/ncu/trsm.log 2>&1
$N -k regex:pack_tiles_kernel -c 1 -o gpurun_out/ncu/pack -f python tools/one_step.py --steps 1 > gpurun_out/ncu/pack.log 2>&1
$N -k regex:potrf_inv_kernel -s 20 -c 1 -o gpurun_out/ncu/potrf -f python tools/one_step.py --steps 1 > gpurun_out/ncu/potrf.log 2>&1
$N -k regex:prefix_kernel -c 1 -o gpurun_out/ncu/prefix -f python tools/one_step.py --steps 1 > gpurun_out/ncu/prefix.log 2>&1
for r in trsm pack potrf prefix; do python tools/ncu_kernel_summary.py gpurun_out/ncu/$r.ncu-rep > gpurun_out/ncu/$r.json 2>&1; done
ls -la gpurun_out/ncu
