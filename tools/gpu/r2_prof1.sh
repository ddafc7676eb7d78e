# Round-2 baseline evidence: K1 gather microbench, attention vs SDPA yardstick, and one ncu pass
# (duration + DRAM bytes + tensor pipe) over every kernel of one Llama-1B step.
O=gpurun_out/r2prof; mkdir -p $O
python tools/bench_gather.py 4 4096 16384 > $O/gather_w4.json 2>&1; echo gather4 $?
python tools/bench_gather.py 2 2048 32768 > $O/gather_w2.json 2>&1; echo gather2 $?
python tools/bench_attn.py > $O/attn_yardstick.jsonl 2>&1; echo attn $?
python tools/profile_step.py llama-1b 4 4096 2 > $O/step_plain.log 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/llama1b_step_metrics.csv python tools/profile_step.py llama-1b 4 4096 2 > $O/ncu_step.log 2>&1; echo ncu_step $?
python tools/bench_gather.py 4 4096 16384 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:gather_samples -s 5 -c 3 --csv --log-file $O/gather_ncu.csv python tools/bench_gather.py 4 4096 16384 > /dev/null 2>&1; echo ncu_gather $?
ls -la $O
