O=gpurun_out/r2pf; mkdir -p $O
python tools/one_attn.py 4 4096 32 8 bwd > $O/attn.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 1 -c 1 -o $O/attn_bwd_1b python tools/one_attn.py 4 4096 32 8 bwd > /dev/null 2>&1; echo a2 $?
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm_swiglu_bwd python tools/one_swiglu_bwd.py > /dev/null 2>&1; echo g $?
python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/llama1b_step_metrics.csv python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1; echo step $?
python tools/profile_step.py gpt2-124m 8 2048 2 > /dev/null 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/gpt2_step_metrics.csv python tools/profile_step.py gpt2-124m 8 2048 2 > /dev/null 2>&1; echo step2 $?
ls -la $O
