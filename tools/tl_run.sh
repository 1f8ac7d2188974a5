mkdir -p gpurun_out
for v in 2 3; do
  B2D_LIB_OVERRIDE=$PWD/paper_2503_04424_b200/lib/libmemdet_bulk$v.so timeout 300 python tools/ldl_tl.py --tag bulk$v --out gpurun_out/ldl_tl_bulk$v.txt > gpurun_out/ldl_tl_bulk$v.log 2>&1
done
timeout 300 python tools/ldl_tl.py --tag bulk4 --out gpurun_out/ldl_tl_bulk4.txt > gpurun_out/ldl_tl_bulk4.log 2>&1
