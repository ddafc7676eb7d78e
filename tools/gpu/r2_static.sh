for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dyn', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
B2S_GEMM_STATIC_K=16384 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('st16k', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
B2S_GEMM_STATIC_K=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stall', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm'])"
done
python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1 && B2S_GEMM_STATIC_K=16384 python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1 && \
B2S_GEMM_STATIC_K=16384 PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/r2_static_step.csv python tools/profile_step.py llama-1b 4 4096 2 > /dev/null 2>&1; echo ncu $?
