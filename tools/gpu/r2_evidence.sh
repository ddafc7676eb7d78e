O=gpurun_out/r2ev; mkdir -p $O
python -m pytest tests/test_guards.py -m gpu -q > $O/guards.log 2>&1; echo guards $?; tail -3 $O/guards.log
python tools/bench_ew.py > $O/bench_ew.jsonl 2> $O/bench_ew.err; echo ew $?
python tools/bench_kernels.py > $O/bench_kernels.jsonl 2> $O/bench_kernels.err; echo kernels $?
python tools/bench_ew.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"norm_|rope|swiglu|xent|adamw|colsum|embed" -c 400 --csv --log-file $O/bench_ew_ncu.csv python tools/bench_ew.py > /dev/null 2>&1; echo ncu $?
