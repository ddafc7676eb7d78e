O=gpurun_out/r2fp; mkdir -p $O
python tools/one_attn.py 4 4096 32 8 bwd > $O/attn.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o $O/attn_fwd_1b python tools/one_attn.py 4 4096 32 8 bwd > /dev/null 2>&1; echo a1 $?
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 1 -c 1 -o $O/attn_bwd_1b python tools/one_attn.py 4 4096 32 8 bwd > /dev/null 2>&1; echo a2 $?
python tools/one_gemm_w13dgrad.py > $O/gemm.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm_w13_dgrad python tools/one_gemm_w13dgrad.py > /dev/null 2>&1; echo g1 $?
python tools/one_swiglu_fwd.py > $O/swf.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm_swiglu_fwd python tools/one_swiglu_fwd.py > /dev/null 2>&1; echo g2 $?
python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/llama1b_step_metrics.csv python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1; echo step $?
python tools/profile_step.py gpt2-124m 8 2048 2 > /dev/null 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/gpt2_step_metrics.csv python tools/profile_step.py gpt2-124m 8 2048 2 > /dev/null 2>&1; echo step2 $?
ls -la $O
