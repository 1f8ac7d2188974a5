mkdir -p gpurun_out
for kc in 1 2 4 8; do
  B2D_REST_KCHUNK=$kc timeout 300 python tools/ldl_tl.py --tag kc$kc --steps 3 --out gpurun_out/ldl_tl_kc$kc.txt > gpurun_out/ldl_tl_kc$kc.log 2>&1
done
