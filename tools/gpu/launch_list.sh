O=gpurun_out/prof; mkdir -p $O
timeout 300 python tools/profile_step.py > $O/step_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/gpt2_step_launches.csv \
    python tools/profile_step.py > $O/ncu1.log 2>&1; echo ncu1=$?
python tools/launch_table.py $O/gpt2_step_launches.csv > $O/gpt2_step_launches.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
    --clock-control none -k regex:gemm_kernel --csv --log-file $O/gemm_dram_tensor_metrics.csv \
    python tools/profile_step.py > $O/ncu2.log 2>&1; echo ncu2=$?
