O=gpurun_out/r2raster; mkdir -p $O
python -m pytest tests/test_gemm.py tests/test_headline_parity.py -m gpu -q -x -k "gemm" > $O/test_gemm.log 2>&1; echo gemm tests $?
for i in 1 2; do
B2S_GEMM_RASTER=mfast python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_mfast_$i.json 2>$O/err; echo mfast $?
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_raster_$i.json 2>$O/err; echo raster $?
done
python bench.py --config gpt2-124m --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_gpt2.json 2>$O/err; echo gpt2 $?
python tools/profile_step.py llama-1b 4 4096 2 > $O/step_plain.log 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $O/llama1b_step_metrics.csv python tools/profile_step.py llama-1b 4 4096 2 > $O/ncu_step.log 2>&1; echo ncu_step $?
