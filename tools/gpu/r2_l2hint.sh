python -m pytest tests/test_gemm.py tests/test_headline_parity.py -m gpu -q -x -k "gemm or two_layer" 2>&1 | tail -1
for i in 1 2; do
B2S_GEMM_L2HINT=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nohint', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hint', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
done
python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1 && \
PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/r2_l2hint_step.csv python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1; echo ncu $?
