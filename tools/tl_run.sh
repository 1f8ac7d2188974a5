mkdir -p gpurun_out
TAG=base python tools/chol_time.py > gpurun_out/chol_ab.txt 2>&1
TAG=skip_potrf B2D_LIB_OVERRIDE=$PWD/paper_2503_04424_b200/lib/libmemdet_skip.so python tools/chol_time.py >> gpurun_out/chol_ab.txt 2>&1
