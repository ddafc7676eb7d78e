O=gpurun_out/r2dsw3; mkdir -p $O
python tools/one_swiglu_bwd.py x > $O/plain.log 2>&1; cat $O/plain.log
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o $O/dsw python tools/one_swiglu_bwd.py > $O/ncu.log 2>&1; echo ncu $?
