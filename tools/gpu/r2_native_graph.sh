python -m pytest tests/test_train_parity.py tests/test_boundary_e2e.py tests/test_headline_parity.py -m gpu -q -x -k "not gemm_headline and not attn_" 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('native', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['gpu_launches'], d['e2e']['value'])"; done
python tools/profile_step.py llama-1b 4 4096 3 > /dev/null 2>&1 && PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_native_launches.csv python tools/profile_step.py llama-1b 4 4096 3 > /dev/null 2>&1; echo ncu $?
