O=gpurun_out/r2epi; mkdir -p $O
timeout 900 python -m pytest tests/test_gemm.py tests/test_guards.py tests/test_attn.py -q -x -m gpu > $O/test.log 2>&1; echo test $?; tail -1 $O/test.log
python tools/one_swiglu_bwd.py
for i in 1 2; do
python bench.py --steps 10 --warmup 4 --no-cpu-baseline > $O/on_$i.json 2>/dev/null
B2S_GEMM_EPI_HINT=0 python bench.py --steps 10 --warmup 4 --no-cpu-baseline > $O/off_$i.json 2>/dev/null
done
python bench.py --config gpt2-124m --steps 10 --warmup 4 --no-cpu-baseline > $O/gpt2_on.json 2>/dev/null
B2S_GEMM_EPI_HINT=0 python bench.py --config gpt2-124m --steps 10 --warmup 4 --no-cpu-baseline > $O/gpt2_off.json 2>/dev/null
for f in $O/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['kernels']['gemm']['ms_per_step'], d['kernels']['attn_bwd']['ms_per_step'])"; done
