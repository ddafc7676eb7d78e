O=gpurun_out/r2attn; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/xu_rate tools/micro/xu_rate.cu && /tmp/xu_rate > $O/xu_rate.txt 2>&1; echo xu $?
python tools/one_attn.py 4 4096 32 8 bwd > $O/one_attn.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o $O/attn_fwd_1b python tools/one_attn.py 4 4096 32 8 bwd > $O/ncu_fwd.log 2>&1; echo fwd $?
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 1 -c 1 -o $O/attn_bwd_1b python tools/one_attn.py 4 4096 32 8 bwd > $O/ncu_bwd.log 2>&1; echo bwd $?
ls -la $O
