O=gpurun_out/r2mn; mkdir -p $O
ncu --set full --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o $O/kk python tools/one_gemm.py 8192 8192 8192 0 0 > $O/kk.log 2>&1; echo $?
ncu --set full --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o $O/mm python tools/one_gemm.py 8192 8192 8192 1 1 > $O/mm.log 2>&1; echo $?
