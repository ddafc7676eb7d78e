O=gpurun_out/r2pf; mkdir -p $O
python tools/profile_step.py llama-1b 4 4096 3 > $O/step_llama.log 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/llama1b_step_metrics.csv python tools/profile_step.py llama-1b 4 4096 3 > /dev/null 2>&1; echo step $?
python tools/profile_step.py gpt2-124m 8 2048 3 > $O/step_gpt2.log 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/gpt2_step_metrics.csv python tools/profile_step.py gpt2-124m 8 2048 3 > /dev/null 2>&1; echo step2 $?
cat $O/step_llama.log $O/step_gpt2.log
